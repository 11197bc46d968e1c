#!/bin/bash
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 3 python tools/sanitize_run.py 2>&1 | grep -v "Host Frame\|Saved host" | head -40
