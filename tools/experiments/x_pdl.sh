mkdir -p gpurun_out; rm -f gpurun_out/x_pdl.txt
for env in "" "DPF_PDL=0"; do
  for c in c2 c3; do
    for prf in chacha20 chacha20_et; do
      env $env timeout 300 python bench.py --config $c --prf $prf --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
      python - "$env" $c $prf <<'PY' >> gpurun_out/x_pdl.txt
import json,sys
l=[x for x in open('/tmp/b.json') if x.startswith('{')]
if not l: print(sys.argv[1:], 'FAIL', open('/tmp/b.err').read()[-300:]); sys.exit()
d=json.loads(l[-1]); r=d['roofline']
print("%-10s %s %-12s qps %9.0f ms %.4f kern %.4f frac %.3f step_frac %.3f e2e %.0f" % (sys.argv[1] or 'pdl', sys.argv[2], sys.argv[3], d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], r['frac_qps'], d['e2e']['value']))
PY
    done
  done
  env $env timeout 300 python tools/batch_sweep.py --log-n 22 --D 64 --B 1 2 4 >> gpurun_out/x_pdl.txt 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python tools/codesign_bench.py --scheme pbr --bins 4 --batches 1 16 256 > gpurun_out/c5_pbr.jsonl 2>&1
timeout 900 python tools/codesign_bench.py --scheme pbr --bins 4 --packed --prf chacha20_et --batches 16 256 1024 > gpurun_out/c5_pbr_et_packed.jsonl 2>&1
