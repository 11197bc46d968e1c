mkdir -p gpurun_out; rm -f gpurun_out/x_pipe.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "server" > gpurun_out/pytest_pipe.txt 2>&1; tail -1 gpurun_out/pytest_pipe.txt
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  python -c "
import json; l=[x for x in open('/tmp/b.json') if x.startswith('{')]; d=json.loads(l[-1]); print('$c', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['value']/d['value'],3))" >> gpurun_out/x_pipe.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/x_pipe.txt
  timeout 600 python bench.py --config $c --prf chacha20_et --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  python -c "
import json; l=[x for x in open('/tmp/b.json') if x.startswith('{')]; d=json.loads(l[-1]); print('$c ET', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['value']/d['value'],3))" >> gpurun_out/x_pipe.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/x_pipe.txt
done
