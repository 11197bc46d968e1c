mkdir -p gpurun_out; O=gpurun_out/sanitizer_r02.txt
echo "# compute-sanitizer over tools/sanitize_run.py (IMAD, tcgen05 single + CTA pair + small-batch Kr mapping, padded D, ET, AES, grouped, PBR), r02 kernels" > $O
echo "== memcheck" >> $O; timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_run.py >> $O 2>&1 | tail -3
echo "== synccheck" >> $O; timeout 1500 compute-sanitizer --tool synccheck python tools/sanitize_run.py >> $O 2>&1
echo "== initcheck" >> $O; timeout 1500 compute-sanitizer --tool initcheck python tools/sanitize_run.py >> $O 2>&1
echo "== racecheck" >> $O; timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_run.py > /tmp/race.txt 2>&1; grep -E "RACECHECK SUMMARY|parity|Error" /tmp/race.txt | sort | uniq -c | head -20 >> $O; grep -A3 "Error: Potential" /tmp/race.txt | head -12 >> $O; python tools/race_classify.py /tmp/race.txt >> $O
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|parity" $O
