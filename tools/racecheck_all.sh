# racecheck, all hazards listed, summarised per kernel / source line
mkdir -p gpurun_out/sanitize2
for c in tiny_cold llama_width odd_groups; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 1000000 python tools/sanitize_cases.py $c > gpurun_out/sanitize2/racecheck_$c.log 2>&1
  echo "rc $? $c" >> gpurun_out/sanitize2/summary.txt
  grep -E "Write Thread|Read Thread" gpurun_out/sanitize2/racecheck_$c.log | sed -E 's/0x[0-9a-f]+/X/g; s/Thread \([0-9,]+\)//; s/\(CUtensorMap.*\)\+X//; s/\(block rank [0-9]\)//' | sort | uniq -c | sort -rn | head -30 >> gpurun_out/sanitize2/summary.txt
  grep SUMMARY gpurun_out/sanitize2/racecheck_$c.log >> gpurun_out/sanitize2/summary.txt
  gzip -f gpurun_out/sanitize2/racecheck_$c.log
done
