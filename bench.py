#!/usr/bin/env python
"""bench.py -- DPF-PIR server throughput (queries/s) on B200, BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

A step = one server's answer to one batch of B DPF keys (BASELINE config c3 by
default: 2^20 x 256 int32 table, B = 256): a1 key ingest, a2 top BFS, a3-a6
the fused expansion x table kernel, a7 the B x D answer; for N > 1 the table is
row-sharded (rank r owns rows [r N/G, (r+1) N/G)) and the partial answers are
summed mod 2^32 by one NCCL reduce to rank 0 -- strong scaling,
the total work per step is fixed.

`value`: keys already in HBM (dpf_eval_batch_wire), timed with CUDA events
over exactly K steps between barriers, max over ranks.  `e2e`: the same through
the host-buffer API (host keys -> pinned staging -> H2D, answer D2H to pinned
host memory every step).  `roofline`: the fused kernel's live per-launch CUDA
event time against the ALU-pipe peak.  `cpu_baseline`:
the CPU oracle (oracle/, test infrastructure) on a bounded sample of the same
keys, which also re-checks bit-exact parity before the line is printed.
`--impl reference`: the oracle alone (the paper has no public GPU code), on the
host cores, same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

# ALU-pipe ops per tree node: ChaCha20 = 320 XOR + 320
# rotate per block (80 quarter rounds; the adds run on the FMA pipe).  AES-128
# (bitsliced, table-free) = the compiled ALU instructions of one node's two
# encryptions + key schedule in this formulation (9 x 411 + 336 + 40 setup;
# Boyar-Peralta S-box = 95 LOP3): a better circuit would lower it.
ALU_OPS_PER_BLOCK = {"chacha20": 640, "aes128": 4075, "chacha20_et": 640}
# leaf rows per tree leaf: early termination (R20) ends the tree at final
# nodes of 16 rows, each converted by one more ChaCha20 block (counter 1).
ET_BITS = {"chacha20": 0, "aes128": 0, "chacha20_et": 4}


def prf_code(dpfpir, name):
    return {"chacha20": dpfpir.DPF_PRF_CHACHA20, "aes128": dpfpir.DPF_PRF_AES128,
            "chacha20_et": dpfpir.DPF_PRF_CHACHA20_ET}[name]
METRIC = "DPF-PIR queries/sec"
UNIT = "queries/s"


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update(hbm_gbs=float(m.get("hbm_gbs", p["hbm_gbs"])), sm_max_mhz=float(m.get("sm_max_mhz", 1965.0)),
                 source="measured (MEASURED_PEAKS.json)")
    return p


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


def make_keys(w, dpfpir, prf=1):
    """B client queries of config w: party-0 keys go to this server (the
    second server is an identical, independent machine)."""
    al = synth.alphas(w.B, w.N, w.seed)
    seeds = synth.gen_seeds(w.B, w.seed)
    pairs = [dpfpir.gen(w.log_n, int(a), 1, s, prf=prf) for a, s in zip(al, seeds)]
    return al, pairs


def oracle_sample(w, keys_wire, T, threads, sample):
    """CPU oracle on `sample` keys with `threads` POSIX threads; returns
    (shares, seconds)."""
    from oracle import oracle as orc
    orc.build()
    okeys = [orc.key_from_wire(bytes(keys_wire[i])) for i in range(sample)]
    t0 = time.perf_counter()
    sh = orc.answer_batch(okeys, T, threads=threads)
    return sh, time.perf_counter() - t0


def cpu_threads():
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(n, 64))


# ---------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    if rank != 0:
        return 0
    w = synth.CONFIGS[args.config]
    from paper_2301_10904_b200 import build as pbuild
    from paper_2301_10904_b200 import dpfpir
    pbuild.build()  # host-side Gen only (client work, outside the timed region)
    prf = prf_code(dpfpir, args.prf)
    _, pairs = make_keys(w, dpfpir, prf)
    wire = dpfpir.keys_to_wire([p[0] for p in pairs])
    T = synth.table(w.N, w.D, w.seed)
    threads = cpu_threads()
    sample = min(w.B, threads)
    times = []
    for i in range(args.warmup + args.steps):
        _, dt = oracle_sample(w, wire, T, threads, sample)
        if i >= args.warmup:
            times.append(dt)
    step = sum(times) / len(times)
    value = sample / step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": w.name + ": " + w.note, "log_n": w.log_n, "N": w.N, "D": w.D, "B": w.B},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": "%d of the %d keys per step (one key per thread), full 2^%d-row table" %
                                   (sample, w.B, w.log_n)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the paper publishes no code; the reference arm is this repo's plain CPU oracle "
                "(oracle/dpf_oracle.c) on the host cores",
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prf", default="chacha20", choices=["chacha20", "aes128", "chacha20_et"],
                    help="tree PRF (chacha20 = the paper's fastest standard PRF, Table 5; aes128 = its baseline; "
                         "chacha20_et = ChaCha20 with early-terminated 16-row leaves, DESIGN.md R20)")
    ap.add_argument("--table", default="auto", choices=["auto", "packed", "rowmajor"],
                    help="packed = limb-packed table + tcgen05 contraction (any D %% 4 == 0, padded to 128-column tiles); rowmajor = IMAD path")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--reduce", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1: sum the row shards' partial answers with one NCCL reduce, or inside the fused "
                         "kernels (every rank red.adds into rank 0's buffer over a CUDA IPC / NVLink mapping)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    import torch
    import torch.distributed as dist
    from paper_2301_10904_b200 import dpfpir, shard

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    G = world
    w = synth.CONFIGS[args.config]
    r0, rows = shard.row_range(w.N, G, rank)
    g = (G - 1).bit_length()  # path levels each rank descends above its subtree(s)

    T_host = synth.table_rows(w.N, w.D, w.seed, r0, r0 + rows)
    T = torch.from_numpy(T_host.view(np.int32)).to(dev)
    use_packed = args.table == "packed" or (args.table == "auto" and w.D <= 1024 and w.B >= 32)
    # server state: the table is re-laid-out once into u8 limb planes (outside every timed region)
    Tp = dpfpir.table_pack(T, r0) if use_packed else None
    torch.cuda.synchronize()
    prf = prf_code(dpfpir, args.prf)
    al, pairs = make_keys(w, dpfpir, prf)
    keys0 = dpfpir.KeyBatch.from_keys([p[0] for p in pairs])
    wire_host = dpfpir.keys_to_wire(keys0)
    wire = torch.from_numpy(wire_host).to(dev)
    ws = torch.empty(dpfpir.serve_workspace_bytes(w.B, w.log_n, rows, w.D), dtype=torch.uint8, device=dev)
    out = torch.empty((w.B, w.D), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    peer = shard.PeerShareReducer(out, dst=0) if (G > 1 and args.reduce == "p2p") else None

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
            shard.reduce_partial_shares(out, dst=0)

    def barrier():
        if G > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    # ---- correctness before timing: both servers' answers reconstruct T[alpha]
    step()
    share0 = dpfpir.as_u32(out) if rank == 0 else None
    keys1 = dpfpir.KeyBatch.from_keys([p[1] for p in pairs])
    out1 = (dpfpir.eval_batch_packed(keys1, Tp, workspace=ws) if use_packed else
            dpfpir.eval_batch_shard(keys1, T, r0, workspace=ws))
    if G > 1:
        shard.reduce_partial_shares(out1, dst=0)
    parity = {}
    if rank == 0:
        recon = dpfpir.reconstruct(share0, dpfpir.as_u32(out1))
        want = np.stack([synth.table_rows(w.N, w.D, w.seed, int(a), int(a) + 1)[0] for a in al])
        parity["reconstruct_all_queries"] = bool(np.array_equal(recon, want))
    barrier()

    # ---- value: device-resident keys, K steps between barriers
    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(_nvsmi_index(local_rank))
    sampler.start()
    dpfpir.kernel_timer_begin(args.steps)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    kernel_ms = dpfpir.kernel_timer_read(args.steps)
    stats = dpfpir.last_eval_stats()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = w.B / (ms_per_step * 1e-3)

    # ---- e2e: host keys in, host answer out, every step
    e2e_steps = args.e2e_steps or max(3, args.steps // 2)
    host_out = torch.empty((w.B, w.D), dtype=torch.int32).pin_memory()

    # G == 1: the graph-captured serving step (dpf_server_*): host wire keys in,
    # host answers out, one graph launch per batch
    server = dpfpir.Server(w.B, w.log_n, Tp if use_packed else T, r0, prf=prf, stream=stream) if G == 1 else None
    host_out_np = host_out.numpy().view(np.uint32)

    def e2e_step():
        if server is not None:
            server.run(wire_host, host_out_np)
            return
        if use_packed:
            dpfpir.eval_batch_packed(keys0, Tp, out=out, workspace=ws, stream=stream)
        else:
            dpfpir.eval_batch_shard(keys0, T, r0, out=out, workspace=ws, stream=stream)
        if G > 1:
            shard.reduce_partial_shares(out, dst=0)
        if rank == 0:
            host_out.copy_(out, non_blocking=True)
        stream.synchronize()

    for _ in range(2):
        e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = w.B / (float(te.item()) / e2e_steps * 1e-3)
    if rank == 0:
        parity["e2e_equals_device_path"] = bool(np.array_equal(host_out.numpy().view(np.uint32), share0))

    # ---- roofline of the dominant kernel (fused eval), live CUDA-event time
    pk = peaks()
    v = ET_BITS[args.prf]
    m = w.log_n - v - stats["frontier_depth"]
    # algorithmic blocks per launch (no padding): the subtrees' internal nodes,
    # plus one Convert block per final node with early termination
    fused_blocks = w.B * ((rows >> v) >> m) * ((1 << m) - 1 + ((1 << m) if v else 0))
    kern_avg_ms = sum(kernel_ms) / len(kernel_ms)
    alu_peak = 148 * 64 * pk["sm_max_mhz"] * 1e6  # ALU-pipe lane-ops/s
    ops_per_block = ALU_OPS_PER_BLOCK[args.prf]
    achieved = ops_per_block * fused_blocks / (kern_avg_ms * 1e-3)
    tree_blocks = (rows - 1 + g) if not v else (2 * (rows >> v) - 1 + g)
    qps_roof = alu_peak / (ops_per_block * tree_blocks)
    hbm_qps_roof = G * pk["hbm_gbs"] * 1e9 * w.B / (4.0 * w.N * w.D)
    traffic = _ncu_traffic(w.name if args.prf == "chacha20" else "%s_%s" % (w.name, args.prf))
    roofline = {
        "bound": "alu", "achieved": achieved * 1e-12, "peak": alu_peak * 1e-12, "unit": "Tops/s",
        "frac": achieved / alu_peak, "traffic": traffic,
        "kernel": "fused_eval_tc_kernel" if use_packed else "fused_eval_kernel", "kernel_ms": kern_avg_ms,
        "kernel_share_of_step": kern_avg_ms / ms_per_step,
        "ops": ("640 ALU-pipe int32 ops (LOP3 xor + SHF rotate) per ChaCha20 block" if args.prf != "aes128" else
                "4075 ALU-pipe ops per bitsliced AES-128 node (2 blocks + key schedule)") +
               " x %d blocks per launch" % fused_blocks,
        "peak_basis": "148 SMs x 64 ALU lanes/clk x %.0f MHz (%s)" % (pk["sm_max_mhz"], pk["source"]),
        "qps_at_prf_roofline": qps_roof, "frac_qps": value / qps_roof, "qps_at_hbm_roofline": hbm_qps_roof,
    }

    # ---- CPU oracle beside it (rank 0, N = 1 only), doubles as a parity sample
    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        T_full = T_host  # G == 1: the whole table
        # bounded sample: chunks of `threads` keys (one per thread) until ~10 s
        # of CPU work or the whole batch; every key is also a parity check
        chunk = min(w.B, max(threads, 8))
        sample, dt, exact = 0, 0.0, True
        while sample < w.B and (sample == 0 or dt < 10.0):
            k = min(chunk, w.B - sample)
            sh, t = oracle_sample(w, wire_host[sample:sample + k], T_full, threads, k)
            exact &= bool(np.array_equal(sh, share0[sample:sample + k]))
            sample += k
            dt += t
        parity["oracle_sample_keys"] = sample
        parity["bit_exact_vs_oracle"] = exact
        cpu = {"value": sample / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": "first %d of the %d party-0 keys, full table, %d threads, %.1f s wall" %
                         (sample, w.B, threads, dt)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": w.name + ": " + w.note, "log_n": w.log_n, "N": w.N, "D": w.D, "B": w.B,
                       "prf": args.prf,
                       "parallelism": ("row-shard x%d + %s" % (G, "NCCL reduce" if args.reduce == "nccl" else
                                       "in-kernel red.add into rank 0 over NVLink (CUDA IPC)")) if G > 1 else "1 GPU",
                       "keys": "device-resident wire keys (dpf_eval_batch_wire%s)" % ("_packed" if use_packed else ""),
                       "table": "limb-packed (dpf_table_pack, tcgen05 kind::i8 contraction)" if use_packed
                       else "row-major int32 (IMAD contraction)",
                       "l2": "no flush: table shard (%d MiB) >= L2 and the path is ALU-bound" %
                             (rows * w.D * 4 >> 20)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(wire_host.nbytes),
                    "d2h_bytes_per_step": w.B * w.D * 4, "api": ("dpf_server_run (CUDA-graph serving step)" if G == 1 else
                            "dpf_eval_batch%s + %sD2H" % ("_packed" if use_packed else "_shard",
                                                          "NCCL reduce + " if G > 1 else ""))},
            "gpu_launches": int(stats["kernels"]) * args.steps,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "parity": parity,
            "plan": stats,
        }
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    if G > 1:
        dist.barrier(device_ids=[local_rank])
        dist.destroy_process_group()
    return 0


def _nvsmi_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [x.strip() for x in vis.split(",") if x.strip()]
        if local_rank < len(ids) and ids[local_rank].isdigit():
            return int(ids[local_rank])
    return local_rank


def _ncu_traffic(config_name: str):
    """DRAM bytes per fused launch from the committed ncu --set full capture
    (profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(config_name, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


if __name__ == "__main__":
    sys.exit(main())
