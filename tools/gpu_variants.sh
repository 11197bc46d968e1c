#!/bin/bash
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_b1.csv python tools/codesign_bench.py --batches 1 --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o /tmp/prof_c5 python tools/codesign_bench.py --batches 1 --steps 2 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_c5.ncu-rep > gpurun_out/ncu_c5_b1.txt 2>&1
python tools/sass_hot.py /tmp/prof_c5.ncu-rep 30 >> gpurun_out/ncu_c5_b1.txt 2>&1
ncu -i /tmp/prof_c5.ncu-rep --page source --csv --print-source sass > /tmp/src.csv 2>/dev/null; python - <<'PY' > gpurun_out/c5_ctx.txt
import csv
rows=list(csv.reader(open('/tmp/src.csv')))
hdr=rows[1]; data=[r for r in rows[2:] if len(r)==len(hdr)]
i_s=hdr.index("Warp Stall Sampling (All Samples)"); i_src=hdr.index("Source"); i_n=hdr.index("Instructions Executed")
val=lambda r: int(r[i_s]) if r[i_s].isdigit() else 0
top=sorted(range(len(data)), key=lambda k:-val(data[k]))[:4]
for k in top:
    print("-----")
    for r in data[max(0,k-14):k+3]: print(val(r), r[0][-5:], r[i_src][:90], r[i_n])
PY
