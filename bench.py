#!/usr/bin/env python
"""bench.py -- DPF-PIR server throughput (queries/s) on B200, BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

`python bench.py --gpus N` with N > 1 and no WORLD_SIZE in the environment
re-launches itself under torch.distributed.run with N ranks (one per GPU);
under torchrun WORLD_SIZE must equal --gpus.

A step = one server's answer to one batch of B DPF keys (BASELINE config c3 by
default: 2^20 x 256 int32 table, B = 256): a1 key ingest, a2 top BFS, a3-a6
the fused expansion x table kernel, a7 the B x D answer; for N > 1 the table is
row-sharded (rank r owns rows [r N/G, (r+1) N/G)) and the partial answers are
summed mod 2^32 by one NCCL reduce to rank 0 -- strong scaling,
the total work per step is fixed.

`value`: keys already in HBM (dpf_eval_batch_wire*), timed with CUDA events
over exactly K steps between barriers, max over ranks; per-step events give
p10/p50/p90.  `e2e`: the same through the host-buffer API (host keys ->
pinned staging -> H2D, answer D2H to pinned host memory every step).
`roofline`: the fused kernel's live per-launch CUDA-event time against the
binding resource (ALU pipe, tensor pipe or HBM).
`cpu_baseline`: the CPU oracle (oracle/, test infrastructure) on a bounded
sample of the same keys.

Parity gates the line: every query must reconstruct T[alpha], a sample of the
device answers must equal the oracle bit-exactly (N > 1: the reduced answers
against the oracle on the whole table, plus an all-0xFFFFFFFF-table case
whose partial answers wrap int32), and the e2e answers must equal the
device-path ones.  Any miss prints the diagnostics to stderr and exits 3
without a JSON line on stdout.

`--impl reference`: the oracle alone (the paper has no public GPU code) on
the host cores: keys from the oracle's own Gen, same metric and config.
"""
from __future__ import annotations

import argparse
import json
import re
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

# ALU-pipe ops per PRF unit.  ChaCha20 = 320 XOR + 320
# rotate per block (80 quarter rounds; the adds run on the FMA pipe).  AES-128
# runs table-driven (S-box/T-table lookups in shared memory), so its bound is
# the lookup count per tree node (aes_lookups_per_node) at one conflict-free
# 32-lane LDS per clock per SM; the bitsliced circuit count
# (aes_alu_ops_per_node) is kept as the table-free alternative's floor.
ALU_OPS_PER_BLOCK = {"chacha20": 640, "chacha20_et": 640}
# leaf rows per tree leaf: early termination (R20) ends the tree at final
# nodes of 16 rows, each converted by one more ChaCha20 block (counter 1).
ET_BITS = {"chacha20": 0, "aes128": 0, "chacha20_et": 4}
PRFS = ("chacha20", "aes128", "chacha20_et")
L2_BYTES = 126 * 1024 * 1024
# Parity-failure hook for the bench contract test (flips one answer word
# before the checks): never set in a measurement.
INJECT_ENV = "DPF_BENCH_INJECT_MISMATCH"
# Test-only: run the N > 1 path with every rank on cuda:0 (gloo, host-side
# collectives) so a one-GPU box exercises it; the line carries "test_mode".
SHARED_GPU_ENV = "DPF_BENCH_SHARED_GPU"

METRIC = "DPF-PIR queries/sec"
UNIT = "queries/s"


def aes_alu_ops_per_node() -> float:
    """Circuit count of one AES-128 tree node (R8/R9: the two blocks 0^120||0
    and 0^120||1 encrypted under the node seed, one shared key schedule),
    independent of this implementation: 2-input bit gates of
    the smallest published circuits, divided by 32 (one 32-bit ALU op applies
    a gate to 32 bit-slices):
      SubBytes    10 rounds x 32 S-boxes (16 bytes x 2 blocks) x 113 gates
                  (Boyar-Matthews-Peralta 2013: 32 AND + 81 XOR/XNOR)
      MixColumns  9 rounds x 8 columns (4 x 2 blocks) x 92 XOR (Maximov 2019)
      AddRoundKey 11 x 256 XOR (128 bits x 2 blocks)
      KeyExpand   10 rounds x (4 S-boxes x 113 + 128 XOR) + popcount(Rcon) XOR
    ShiftRows and RotWord are wiring (free in a circuit)."""
    rcon = (0x01, 0x02, 0x04, 0x08, 0x10, 0x20, 0x40, 0x80, 0x1B, 0x36)
    sbox = 113
    gates = (10 * 32 * sbox + 9 * 8 * 92 + 11 * 256 + 10 * (4 * sbox + 128) + sum(bin(r).count("1") for r in rcon))
    return gates / 32.0


def aes_lookups_per_node() -> int:
    """Distinct S-box evaluations of one AES-128 tree node (R8/R9: blocks
    0^120||0 and 0^120||1 under the node seed, one shared key schedule), each
    one table read in any table-driven AES (FIPS-197 5.1.1 SubBytes; the
    T-table form folds ShiftRows/MixColumns into the same read, 5.1.2-5.1.3):
      SubBytes    16 bytes x 2 blocks per round, minus the inputs the two
                  blocks share: in round 1 their states (key XOR plaintext)
                  differ in byte 15 only (16 + 1 distinct), in round 2 in
                  column 0 only -- round 1's output column 0 (16 + 4); from
                  round 3 on MixColumns has spread the difference (32 each)
      KeyExpand   10 rounds x 4 (SubWord)
    = 17 + 20 + 8 x 32 + 40 = 333."""
    return (16 + 1) + (16 + 4) + 8 * 32 + 10 * 4


AES_LOOKUPS_PER_NODE = aes_lookups_per_node()


def prf_code(dpfpir, name):
    return {"chacha20": dpfpir.DPF_PRF_CHACHA20, "aes128": dpfpir.DPF_PRF_AES128,
            "chacha20_et": dpfpir.DPF_PRF_CHACHA20_ET}[name]


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update(hbm_gbs=float(m.get("hbm_gbs", p["hbm_gbs"])), bf16_tflops=float(m.get("bf16_tflops", 1590.0)),
                 sm_max_mhz=float(m.get("sm_max_mhz", 1965.0)), source="measured (MEASURED_PEAKS.json)")
    return p


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_threads():
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(n, 64))


def workload_config(w, prf: str, gpus: int) -> dict:
    """The workload both arms run (identical dicts: the driver compares them)."""
    rows = w.N // gpus
    return {"workload": w.name + ": " + w.note, "log_n": w.log_n, "N": w.N, "D": w.D, "B": w.B, "prf": prf,
            "parallelism": "1 GPU" if gpus == 1 else "row-shard x%d, answers summed mod 2^32 at rank 0" % gpus,
            "l2": ("no flush: the table shard (%d MiB) exceeds L2 (126 MiB) and the path is ALU-bound" %
                   (rows * w.D * 4 >> 20)) if rows * w.D * 4 > L2_BYTES else
                  "L2 flushed between timed steps (256 MiB write; table shard %d MiB < L2)" % (rows * w.D * 4 >> 20)}


def percentiles(xs):
    a = np.asarray(xs, np.float64)
    return {"p10": float(np.percentile(a, 10)), "p50": float(np.percentile(a, 50)),
            "p90": float(np.percentile(a, 90))}


def parity_ok(parity: dict) -> bool:
    """Every boolean flag must hold (and there must be at least one)."""
    flags = [v for v in parity.values() if isinstance(v, bool)]
    return bool(flags) and all(flags)


def emit(line: dict, parity: dict) -> int:
    """Print the JSON line only when parity holds; otherwise stderr + rc 3."""
    if not parity_ok(parity):
        sys.stderr.write("bench.py: PARITY FAILURE, no result line: %s\n" % json.dumps(parity))
        sys.stderr.write(json.dumps(line) + "\n")
        return 3
    print(json.dumps(line), flush=True)
    return 0


def free_port() -> int:
    s = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn(n: int, argv) -> int:
    """Re-launch this script with n ranks under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-lms", "50", "-f", self.path], stdout=subprocess.DEVNULL,
                                         stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8 or not parts[0].isdigit() or int(parts[0]) != self.idx:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for n, v in zip(names, parts[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def oracle_answers(okeys, T, threads):
    """CPU oracle answers for oracle keys with `threads` POSIX threads;
    returns (shares, seconds)."""
    from oracle import oracle as orc
    orc.build()
    t0 = time.perf_counter()
    sh = orc.answer_batch(okeys, T, threads=threads)
    return sh, time.perf_counter() - t0


def oracle_keys_from_wire(wire_rows):
    from oracle import oracle as orc
    orc.build()
    return [orc.key_from_wire(bytes(r)) for r in wire_rows]


# ---------------------------------------------------------------------- reference arm

def run_reference(args, rank):
    """The oracle alone on the host cores (the paper publishes no code): keys
    from the oracle's Gen with the same seeds as the GPU arm (byte-identical
    keys, tests/test_abi.py), full table, bounded per-step sample."""
    if rank != 0:
        return 0
    from oracle import oracle as orc
    orc.build()
    w = synth.CONFIGS[args.config]
    code = {"chacha20": orc.PRF_CHACHA20, "aes128": orc.PRF_AES128, "chacha20_et": orc.PRF_CHACHA20_ET}[args.prf]
    al = synth.alphas(w.B, w.N, w.seed)
    seeds = synth.gen_seeds(w.B, w.seed)
    T = synth.table(w.N, w.D, w.seed)
    threads = cpu_threads()
    sample = min(w.B, threads)
    okeys = [orc.gen(w.log_n, int(a), 1, s, prf=code)[0] for a, s in zip(al[:sample], seeds[:sample])]
    times = []
    for i in range(args.warmup + args.steps):
        _, dt = oracle_answers(okeys, T, threads)
        if i >= args.warmup:
            times.append(dt)
    step = sum(times) / len(times)
    value = sample / step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(w, args.prf, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu": cpu_model(),
                         "sample": "%d of the %d keys per step (one key per thread), full 2^%d-row table" %
                                   (sample, w.B, w.log_n)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "latency_ms": percentiles([t * 1e3 for t in times]),
        "note": "the paper publishes no code; the reference arm is this repo's plain CPU oracle "
                "(oracle/dpf_oracle.c, its own Gen) on the host cores",
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- our arm

def parse(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prf", default="chacha20", choices=list(PRFS),
                    help="tree PRF (chacha20 = the paper's fastest standard PRF, Table 5; aes128 = its baseline; "
                         "chacha20_et = ChaCha20 with early-terminated 16-row leaves, DESIGN.md R20)")
    ap.add_argument("--table", default="auto", choices=["auto", "packed", "rowmajor"],
                    help="packed = limb-packed table + tcgen05 contraction (any D %% 4 == 0, padded to 128-column "
                         "tiles); rowmajor = IMAD path")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--reduce", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1: sum the row shards' partial answers with one NCCL reduce, or inside the fused "
                         "kernels (every rank red.adds into rank 0's buffer over a CUDA IPC / NVLink mapping)")
    ap.add_argument("--dry-env", action="store_true", help=argparse.SUPPRESS)  # launch-contract test hook
    return ap.parse_args(argv)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1:
            return spawn(args.gpus, argv)
        world = 1
    else:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            raise SystemExit("bench.py: WORLD_SIZE=%d but --gpus %d" % (world, args.gpus))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_env:
        # one write(2) per line: atomic on a pipe shared by the ranks
        os.write(1, (json.dumps({"rank": rank, "world": world, "local_rank": local_rank,
                                 "master_addr": os.environ.get("MASTER_ADDR")}) + "\n").encode())
        return 0
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"
    return run_ours(args, rank, world, local_rank)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2301_10904_b200 import dpfpir, shard

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    # Test mode for the N > 1 code path on a one-GPU box (tests/test_bench_gpu.py):
    # every rank on cuda:0, a gloo group, collectives through host copies.  The
    # line says so ("test_mode"); it is never a measurement.
    shared_gpu = os.environ.get(SHARED_GPU_ENV) == "1"
    if shared_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def host_coll(t, fn):
        if not shared_gpu:
            return fn(t)
        h = t.cpu()
        fn(h)
        t.copy_(h)
        return t

    def reduce0(t):  # the one exchange step: partial answers summed mod 2^32 at rank 0
        return host_coll(t, lambda x: shard.reduce_partial_shares(x, dst=0))
    G = world
    w = synth.CONFIGS[args.config]
    r0, rows = shard.row_range(w.N, G, rank)
    g = (G - 1).bit_length()  # path levels each rank descends above its subtree(s)
    inject = os.environ.get(INJECT_ENV) == "1"

    T_host = synth.table_rows(w.N, w.D, w.seed, r0, r0 + rows)
    T = torch.from_numpy(T_host.view(np.int32)).to(dev)
    use_packed = args.table == "packed" or (args.table == "auto" and w.D <= 1024 and w.B >= 32)
    # server state: the table is re-laid-out once into u8 limb planes (outside every timed region)
    Tp = dpfpir.table_pack(T, r0) if use_packed else None
    torch.cuda.synchronize()
    prf = prf_code(dpfpir, args.prf)
    al = synth.alphas(w.B, w.N, w.seed)
    seeds = synth.gen_seeds(w.B, w.seed)
    pairs = [dpfpir.gen(w.log_n, int(a), 1, s, prf=prf) for a, s in zip(al, seeds)]
    keys0 = dpfpir.KeyBatch.from_keys([p[0] for p in pairs])
    wire_host = dpfpir.keys_to_wire(keys0)
    wire = torch.from_numpy(wire_host).to(dev)
    ws = torch.empty(dpfpir.serve_workspace_bytes(w.B, w.log_n, rows, w.D), dtype=torch.uint8, device=dev)
    out = torch.empty((w.B, w.D), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    peer = shard.PeerShareReducer(out, dst=0) if (G > 1 and args.reduce == "p2p") else None
    flush_l2 = rows * w.D * 4 <= L2_BYTES
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_l2 else None

    def step():
        if peer is not None:  # fused reduction: accumulate into rank 0's answers
            peer.begin()
            dpfpir.eval_batch_wire_ex(wire, w.log_n, Tp if use_packed else T, r0, rows, w.D, peer.ptr,
                                      dpfpir.DPF_EVAL_ACCUMULATE, ws, stream=stream, prf=prf, packed=use_packed)
            peer.finish()
            return
        if use_packed:
            dpfpir.eval_batch_wire_packed(wire, w.log_n, Tp, out=out, workspace=ws, stream=stream, prf=prf)
        else:
            dpfpir.eval_batch_wire(wire, w.log_n, T, r0, out=out, workspace=ws, stream=stream, prf=prf)
        if G > 1:
            reduce0(out)

    def barrier():
        if G > 1:
            if shared_gpu:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    # ---- correctness before timing: both servers' answers reconstruct T[alpha]
    step()
    barrier()
    share0 = dpfpir.as_u32(out) if rank == 0 else None
    if share0 is not None and inject:
        share0[0, 0] ^= 1
    keys1 = dpfpir.KeyBatch.from_keys([p[1] for p in pairs])
    out1 = (dpfpir.eval_batch_packed(keys1, Tp, workspace=ws) if use_packed else
            dpfpir.eval_batch_shard(keys1, T, r0, workspace=ws))
    if G > 1:
        reduce0(out1)
    parity = {}
    if rank == 0:
        recon = dpfpir.reconstruct(share0, dpfpir.as_u32(out1))
        want = np.stack([synth.table_rows(w.N, w.D, w.seed, int(a), int(a) + 1)[0] for a in al])
        parity["reconstruct_all_queries"] = bool(np.array_equal(recon, want))
    if G > 1:
        parity.update(wrap_check(args, dpfpir, shard, reduce0, G, rank, dev, use_packed, prf, inject))
    barrier()

    # ---- value: device-resident keys, K steps between barriers
    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(_nvsmi_index(local_rank))
    sampler.start()
    dpfpir.kernel_timer_begin(args.steps)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(args.steps):
        if scrub is not None:
            scrub.fill_(i & 0xFF)  # L2 flush between timed steps (outside the per-step events)
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    ev1.record(stream)
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    region_ms = ev0.elapsed_time(ev1)
    kernel_ms = dpfpir.kernel_timer_read(args.steps)
    stats = dpfpir.last_eval_stats()
    t = torch.tensor([region_ms if scrub is None else sum(step_ms)] + step_ms, dtype=torch.float64, device=dev)
    if G > 1:
        host_coll(t, lambda x: dist.all_reduce(x, op=dist.ReduceOp.MAX))
    tl = t.cpu().tolist()
    ms_per_step = tl[0] / args.steps
    lat = percentiles(tl[1:])
    value = w.B / (ms_per_step * 1e-3)

    # ---- e2e: host keys in, host answer out, every step
    e2e_steps = args.e2e_steps or max(3, args.steps // 2)
    host_out = torch.empty((w.B, w.D), dtype=torch.int32).pin_memory()
    # G == 1: the graph-captured serving step (dpf_server_*): host wire keys in,
    # host answers out, one graph launch per batch
    # (pipelined: 2 batches in flight, each step still uploads its keys and
    # downloads its answers; consecutive steps overlap, as in serving)
    depth = 2
    server = (dpfpir.Server(w.B, w.log_n, Tp if use_packed else T, r0, prf=prf, stream=stream, depth=depth)
              if G == 1 else None)
    host_out_np = host_out.numpy().view(np.uint32)
    in_flight = [0]

    def e2e_step():
        if server is not None:
            if in_flight[0] == depth:
                server.collect(host_out_np)
                in_flight[0] -= 1
            server.submit(wire_host)
            in_flight[0] += 1
            return
        if use_packed:
            dpfpir.eval_batch_packed(keys0, Tp, out=out, workspace=ws, stream=stream)
        else:
            dpfpir.eval_batch_shard(keys0, T, r0, out=out, workspace=ws, stream=stream)
        if G > 1:
            reduce0(out)
        if rank == 0:
            host_out.copy_(out, non_blocking=True)
        stream.synchronize()

    for _ in range(2):
        e2e_step()
    while server is not None and in_flight[0]:  # warm-up batches collected before timing
        server.collect(host_out_np)
        in_flight[0] -= 1
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    while server is not None and in_flight[0]:  # drain: every timed step's answers are on the host
        server.collect(host_out_np)
        in_flight[0] -= 1
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if G > 1:
        host_coll(te, lambda x: dist.all_reduce(x, op=dist.ReduceOp.MAX))
    e2e_value = w.B / (float(te.item()) / e2e_steps * 1e-3)
    if rank == 0:
        e2e_ans = host_out.numpy().view(np.uint32).copy()
        if inject:
            e2e_ans[0, 0] ^= 1
        parity["e2e_equals_device_path"] = bool(np.array_equal(e2e_ans, share0))

    roofline = roofline_of(args, w, rows, g, G, stats, kernel_ms, ms_per_step, value, use_packed)

    # ---- CPU oracle beside it (rank 0): the parity sample; timed only at N = 1
    cpu = None
    if rank == 0:
        cpu, sample_parity = oracle_leg(args, w, wire_host, share0, T_host if G == 1 else None, G)
        parity.update(sample_parity)
    if G > 1:
        barrier()

    rc = 0
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": workload_config(w, args.prf, G),
            "impl_detail": {
                "reduce": "none" if G == 1 else ("one NCCL reduce (int32 SUM)" if args.reduce == "nccl" else
                                                 "in-kernel red.add.sys into rank 0 over NVLink (CUDA IPC)"),
                "keys": "device-resident wire keys (dpf_eval_batch_wire%s)" % ("_packed" if use_packed else ""),
                "table": "limb-packed (dpf_table_pack, tcgen05 kind::i8 contraction)" if use_packed
                else "row-major int32 (IMAD contraction)"},
            "latency_ms": lat,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(wire_host.nbytes),
                    "d2h_bytes_per_step": w.B * w.D * 4, "api": ("dpf_server_submit/collect (CUDA-graph serving steps, 2 in flight)" if G == 1 else
                            "dpf_eval_batch%s + %sD2H" % ("_packed" if use_packed else "_shard",
                                                          "NCCL reduce + " if G > 1 else ""))},
            "gpu_launches": int(stats["kernels"]) * args.steps,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "parity": parity,
            "plan": stats,
        }
        if shared_gpu:
            line["test_mode"] = "all ranks on cuda:0, gloo, host-side collectives (not a measurement)"
        rc = emit(line, parity)
    if peer is not None:
        peer.close()
    if G > 1:
        flag = torch.tensor([rc], dtype=torch.int32, device=dev)
        host_coll(flag, lambda x: dist.broadcast(x, src=0))
        rc = int(flag.item())
        barrier()
        dist.destroy_process_group()
    return rc


def wrap_check(args, dpfpir, shard, reduce0, G, rank, dev, use_packed, prf, inject):
    """N > 1: an all-0xFFFFFFFF table of 2^12 rows, row-sharded like the real
    one, 32 keys with random beta: each rank's partial answers are (minus) sums
    of leaf shares, so their int32 sum overflows in about half the words.  The
    reduced answers must equal the oracle on the whole table bit-exactly, which
    proves the reduce is addition mod 2^32 on this box's NCCL / NVLink path."""
    import torch
    n, N, D, B = 12, 1 << 12, 128, 32
    a0, cnt = shard.row_range(N, G, rank)
    Tw = torch.full((cnt, D), -1, dtype=torch.int32, device=dev)
    Twp = dpfpir.table_pack(Tw, a0) if use_packed else None
    al = synth.alphas(B, N, 0x3A9)
    be = synth.betas(B, 0x3A9, random=True)
    keys = [dpfpir.gen(n, int(a), int(b), s, prf=prf)[0] for a, b, s in zip(al, be, synth.gen_seeds(B, 0x3A9))]
    kb = dpfpir.KeyBatch.from_keys(keys)
    outw = torch.empty((B, D), dtype=torch.int32, device=dev)
    if args.reduce == "p2p":
        pr = shard.PeerShareReducer(outw, dst=0)
        wire = torch.from_numpy(dpfpir.keys_to_wire(kb)).to(dev)
        wsw = torch.empty(dpfpir.eval_workspace_bytes(B, n, cnt, D), dtype=torch.uint8, device=dev)
        pr.begin()
        dpfpir.eval_batch_wire_ex(wire, n, Twp if use_packed else Tw, a0, cnt, D, pr.ptr, dpfpir.DPF_EVAL_ACCUMULATE,
                                  wsw, prf=prf, packed=use_packed)
        pr.finish()
        pr.close()
    else:
        if use_packed:
            dpfpir.eval_batch_packed(kb, Twp, out=outw)
        else:
            dpfpir.eval_batch_shard(kb, Tw, a0, out=outw)
        reduce0(outw)
    torch.cuda.synchronize()
    if rank != 0:
        return {}
    from oracle import oracle as orc
    got = dpfpir.as_u32(outw)
    if inject:
        got[0, 0] ^= 1
    okeys = oracle_keys_from_wire(dpfpir.keys_to_wire(kb))
    ones = np.full((N, D), 0xFFFFFFFF, np.uint32)
    want = orc.answer_batch(okeys, ones, threads=cpu_threads())
    # how many answer words overflow int32 when the per-rank partials are summed
    parts = [orc.answer_batch(okeys, ones[r0:r0 + c], row_begin=r0, threads=cpu_threads())
             for r0, c in (shard.row_range(N, G, r) for r in range(G))]
    s = sum(p.view(np.int32).astype(np.int64) for p in parts)
    wraps = int(np.count_nonzero((s < -(1 << 31)) | (s >= (1 << 31))))
    return {"wrap_reduce_exact": bool(np.array_equal(got, want)), "wrap_reduce_words_overflowing": wraps,
            "wrap_case_exercised": wraps > 0}


def oracle_leg(args, w, wire_host, share0, T_full, G):
    """rank 0.  N = 1: the CPU oracle on chunks of one key per host thread until
    ~10 s of CPU work or the whole batch (every key is a parity check), plus one
    key single-threaded -> cpu_baseline.  N > 1: a sample of the reduced
    answers against the oracle on the whole table (regenerated here with
    synth), untimed (cpu_baseline is rank 0 at N = 1 only)."""
    parity = {}
    threads = cpu_threads()
    if G > 1:
        T_all = synth.table(w.N, w.D, w.seed)
        k = min(w.B, max(4, min(threads, 8 if w.log_n >= 24 else threads)))
        sh, _ = oracle_answers(oracle_keys_from_wire(wire_host[:k]), T_all, min(threads, k))
        parity["oracle_sample_keys"] = k
        parity["bit_exact_vs_oracle"] = bool(np.array_equal(sh, share0[:k]))
        return None, parity
    if args.no_cpu_baseline:
        sh, _ = oracle_answers(oracle_keys_from_wire(wire_host[:1]), T_full, 1)
        parity["oracle_sample_keys"] = 1
        parity["bit_exact_vs_oracle"] = bool(np.array_equal(sh, share0[:1]))
        return None, parity
    chunk = min(w.B, max(threads, 8))
    sample, dt, exact = 0, 0.0, True
    while sample < w.B and (sample == 0 or dt < 10.0):
        k = min(chunk, w.B - sample)
        sh, t = oracle_answers(oracle_keys_from_wire(wire_host[sample:sample + k]), T_full, threads)
        exact &= bool(np.array_equal(sh, share0[sample:sample + k]))
        sample += k
        dt += t
    # one key on one thread (the paper's 1-thread CPU column)
    sh1, t1 = oracle_answers(oracle_keys_from_wire(wire_host[w.B - 1:w.B]), T_full, 1)
    exact &= bool(np.array_equal(sh1, share0[w.B - 1:w.B]))
    parity["oracle_sample_keys"] = min(w.B, sample + 1)
    parity["bit_exact_vs_oracle"] = exact
    cpu = {"value": sample / dt, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu": cpu_model(),
           "single_thread_value": 1.0 / t1,
           "sample": "first %d of the %d party-0 keys, full table, %d threads, %.1f s wall; single thread: "
                     "key %d alone, %.2f s" % (sample, w.B, threads, dt, w.B - 1, t1)}
    return cpu, parity


def tc_smem_operand_bytes(rows: int, D: int, B: int, keys_per_tile: int, pair: bool) -> float:
    """Shared-memory traffic of the tcgen05 limb contraction for one table pass
    per key tile (DESIGN.md §8 "Entry-size sweep"): per key tile of N =
    keys_per_tile keys, 32-row K-chunk and 128-column d-tile, the 10 limb MMAs
    each read the A tile (128 x 32 B) and this CTA's B columns (N, or N/2 for
    a CTA pair, x 32 B), and the T ring takes the 16 KB limb-packed entry once.
    N is fixed by the 512 TMEM columns (4 limb accumulators x d-tiles x N),
    so at large D the table re-streams once per N keys; this bound (at
    128 B/clk/SM) is what binds early termination above 1 KiB entries."""
    n_kt = -(-B // keys_per_tile)
    n_cc = -(-rows // 32)
    n_dt = -(-D // 128)
    n_cta = keys_per_tile // 2 if pair else keys_per_tile
    return float(n_kt) * n_cc * n_dt * (10 * (4096 + 32 * n_cta) + 16384)


def roofline_of(args, w, rows, g, G, stats, kernel_ms, ms_per_step, value, use_packed):
    """The dominant (fused) kernel against whichever resource binds it:
    algorithmic work per launch / that resource's peak, the largest of
      alu    = ALU-pipe ops of the PRF blocks (640 per ChaCha20 block)
                                                      / 148 x 64 lanes x clock
      smem   = AES-128: table lookups of the PRF nodes (333 per node)
                                                      / 148 x 32 lanes x clock
               (one conflict-free LDS.32 per clock per SM)
      tensor = 10 u8 limb MACs x 2 ops per (key, row, column) of the
               contraction (tcgen05 path)             / 2 x the measured bf16
               dense peak (int8 = fp8 rate = 2 x bf16, B200_PROFILING.md)
      hbm    = the table shard read once              / the measured copy BW
    frac = (that lower bound) / the live per-launch time."""
    pk = peaks()
    v = ET_BITS[args.prf]
    m = w.log_n - v - stats["frontier_depth"]
    # algorithmic blocks per launch (no padding): the subtrees' internal nodes,
    # plus one Convert block per final node with early termination
    fused_blocks = w.B * ((rows >> v) >> m) * ((1 << m) - 1 + ((1 << m) if v else 0))
    kern_avg_ms = sum(kernel_ms) / len(kernel_ms)
    aes = args.prf == "aes128"
    # the PRF's binding unit: ALU-pipe ops (ChaCha20) or SMEM table lookups (AES)
    prf_res = "smem" if aes else "alu"
    alu_peak = 148 * (32 if aes else 64) * pk["sm_max_mhz"] * 1e6  # lanes/s of that unit
    ops_per_block = AES_LOOKUPS_PER_NODE if aes else ALU_OPS_PER_BLOCK[args.prf]
    alu_work = ops_per_block * fused_blocks
    tensor_peak = 2.0 * pk["bf16_tflops"] * 1e12
    tensor_work = 2.0 * 10 * w.B * rows * w.D if use_packed else 0.0
    hbm_peak = pk["hbm_gbs"] * 1e9
    hbm_work = 4.0 * rows * w.D
    smem_peak = 148 * 128 * pk["sm_max_mhz"] * 1e6  # B/s
    smem_work = (tc_smem_operand_bytes(rows, w.D, w.B, stats["keys_per_tile"], bool((stats.get("kernel_id", 0) >> 1) & 1))
                 if use_packed else 0.0)
    bounds = {prf_res: alu_work / alu_peak, "tensor": tensor_work / tensor_peak, "hbm": hbm_work / hbm_peak}
    if use_packed:
        bounds["smem_operands"] = smem_work / smem_peak
    bound = max(bounds, key=bounds.get)
    work, peak, unit = {prf_res: (alu_work, alu_peak, "T lookups/s" if aes else "Tops/s"),
                        "smem_operands": (smem_work, smem_peak, "GB/s"),
                        "tensor": (tensor_work, tensor_peak, "TOPS (int8)"),
                        "hbm": (hbm_work, hbm_peak, "GB/s")}[bound]
    scale = 1e-9 if bound in ("hbm", "smem_operands") else 1e-12
    achieved = work / (kern_avg_ms * 1e-3)
    tree_blocks = (rows - 1 + g) if not v else (2 * (rows >> v) - 1 + g)
    qps_roof = min(alu_peak / (ops_per_block * tree_blocks),
                   w.B / max(bounds["tensor"], bounds["hbm"], bounds.get("smem_operands", 0.0), 1e-30))
    from paper_2301_10904_b200 import dpfpir
    timed_kernel = dpfpir.kernel_name(stats.get("kernel_id", 0))
    traffic, traffic_kernel = _ncu_traffic(w.name if args.prf == "chacha20" else "%s_%s" % (w.name, args.prf))
    if traffic is not None and traffic_kernel != timed_kernel:
        traffic = None  # the capture is of another kernel instantiation than the one just timed
    return {
        "bound": bound, "achieved": achieved * scale, "peak": peak * scale, "unit": unit,
        "frac": achieved / peak, "traffic": traffic, "traffic_kernel": traffic_kernel, "timed_kernel": timed_kernel,
        "bounds_ms": {k: v_ * 1e3 for k, v_ in bounds.items()},
        "kernel": "fused_eval_tc_kernel" if use_packed else "fused_eval_kernel", "kernel_ms": kern_avg_ms,
        "kernel_share_of_step": kern_avg_ms / ms_per_step,
        "ops": ("%d SMEM table lookups per AES-128 node (S-box evaluations, DESIGN.md §7) x %d per launch" %
                (ops_per_block, fused_blocks) if aes else
                "%g ALU-pipe ops per ChaCha20 block (LOP3 xor + SHF rotate) x %d per launch" %
                (ops_per_block, fused_blocks)),
        "peak_basis": {prf_res: ("148 SMs x 32 LDS lanes/clk x %.0f MHz" if aes else
                                 "148 SMs x 64 ALU lanes/clk x %.0f MHz") % pk["sm_max_mhz"],
                       "smem_operands": "148 SMs x 128 B/clk x %.0f MHz (B300_MICROARCH.md smem crossbar)" %
                                        pk["sm_max_mhz"],
                       "tensor": "2 x %.1f TFLOP/s bf16 (%s)" % (pk["bf16_tflops"], pk["source"]),
                       "hbm": "%.0f GB/s (%s)" % (pk["hbm_gbs"], pk["source"])},
        "qps_at_roofline": qps_roof, "frac_qps": value / qps_roof,
        "table_bytes_streamed": 4.0 * rows * (((w.D + 127) // 128 * 128) if use_packed else w.D) *
                                max(1, -(-w.B // max(1, stats["keys_per_tile"]))),
    }


def _nvsmi_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [x.strip() for x in vis.split(",") if x.strip()]
        if local_rank < len(ids) and ids[local_rank].isdigit():
            return int(ids[local_rank])
    return local_rank


def _ncu_traffic(config_name: str):
    """(DRAM bytes per fused launch, captured kernel template) from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or (None,
    None).  The caller drops the bytes when the template differs from the
    kernel the run just timed."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            e = json.load(f).get(config_name, {})
    except (OSError, ValueError):
        return None, None
    kern = e.get("kernel")
    if kern:  # ncu prints "void ns::fused_eval_tc_kernel<ns::PrfChacha, 16, 3, 4, 1, 0>(ns::TcParams)"
        kern = re.sub(r"\(.*$", "", kern.replace("void ", "").replace("dpfpir::dev::", "").replace("dpfpir::", "")).strip()
        kern = kern.replace("true", "1").replace("false", "0")
    return e.get("dram_bytes_per_launch"), kern


if __name__ == "__main__":
    sys.exit(main())
