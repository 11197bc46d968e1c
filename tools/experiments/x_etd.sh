mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum --clock-control none -k regex:fused -s 1 -c 1 --csv python tools/prof_one.py --D 1024 --B 256 --iters 2 > gpurun_out/etd_std1024.csv 2>&1
cat > /tmp/p1.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_2301_10904_b200 import dpfpir
n, N, D, B = 20, 1 << 20, int(sys.argv[1]), 256
keys = [dpfpir.gen(n, int(x), 1, s, prf=3)[0] for x, s in zip(synth.alphas(B, N, 1), synth.gen_seeds(B, 1))]
wire = torch.from_numpy(dpfpir.keys_to_wire(keys)).cuda()
pk = dpfpir.table_pack(torch.from_numpy(synth.table(N, D, 7).view(np.int32)).cuda())
for _ in range(2): dpfpir.eval_batch_wire_packed(wire, n, pk, prf=3)
torch.cuda.synchronize(); print(dpfpir.last_eval_stats())
PY
for d in 512 1024; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum --clock-control none -k regex:fused -s 1 -c 1 --csv python /tmp/p1.py $d > gpurun_out/etd_et$d.csv 2>&1
done
