#!/usr/bin/env bash
# compute-sanitizer passes over the hand-written sm_100a kernels
# (tools/sanitize_cases.py) and the peer-memory allreduce (two processes on
# one GPU). Logs go to gpurun_out/sanitize/; copy the summaries to profiles/.
#   gpurun -- bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p "$OUT"
CS=${CS:-compute-sanitizer}
run() {  # tool case timeout
  local tool=$1 case=$2 to=$3
  echo "== $tool $case" | tee -a "$OUT/summary.txt"
  timeout "$to" $CS --tool "$tool" --error-exitcode 99 --print-limit 50 ${EXTRA:-} \
    python tools/sanitize_cases.py "$case" > "$OUT/${tool}_${case}.log" 2>&1
  local rc=$?
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case .* ok" "$OUT/${tool}_${case}.log" | tail -3 | tee -a "$OUT/summary.txt"
  echo "rc $rc" | tee -a "$OUT/summary.txt"
}
for c in tiny_cold llama_width odd_groups; do
  run memcheck "$c" 600
done
for c in tiny_cold llama_width odd_groups; do
  run synccheck "$c" 600
done
for c in tiny_cold llama_width; do
  EXTRA="--racecheck-report all" run racecheck "$c" 900
done
run initcheck tiny_cold 600
# peer allreduce: both processes under memcheck
echo "== memcheck peer allreduce (2 processes)" | tee -a "$OUT/summary.txt"
timeout 600 $CS --tool memcheck --target-processes all --error-exitcode 99 \
  python -m pytest tests/test_peer_allreduce.py -x -q -m gpu > "$OUT/memcheck_peer.log" 2>&1
echo "rc $?" | tee -a "$OUT/summary.txt"
grep -E "ERROR SUMMARY|passed|failed" "$OUT/memcheck_peer.log" | tail -5 | tee -a "$OUT/summary.txt"
