# A/B driver: "label:ENV=... " variants x one bench config, one summary line each
# (tuning only; a variant that breaks parity is marked PARITY-FAIL, its timing
# is still read from the diagnostic line bench.py writes to stderr).
# usage: bash tools/ab.sh "<bench args>" "label:ENV=1 ENV2=2" "label2:" ...
args="$1"; shift
mkdir -p gpurun_out
for v in "$@"; do
  label="${v%%:*}"; envs="${v#*:}"
  env $envs timeout 600 python bench.py $args --no-cpu-baseline > /tmp/ab_out.txt 2>&1
  rc=$?
  python - "$label" "$args" "$rc" <<'EOF' | tee -a gpurun_out/ab.txt
import json, sys
label, args, rc = sys.argv[1], sys.argv[2], int(sys.argv[3])
lines = [l for l in open("/tmp/ab_out.txt") if l.startswith("{")]
if not lines:
    print("%-24s %s FAILED rc=%d %s" % (label, args, rc, open("/tmp/ab_out.txt").read()[-300:]))
    sys.exit(0)
d = json.loads(lines[-1]); r = d["roofline"]
print("%-24s %-46s qps %9.0f  ms %.4f  kern %.4f  frac %.4f  step_frac %.4f  p50 %.4f%s" % (
    label, args, d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"], r["frac_qps"], d["latency_ms"]["p50"],
    "" if rc == 0 else "  PARITY-FAIL(rc=%d)" % rc))
EOF
done
