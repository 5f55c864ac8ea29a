#!/bin/bash
# compute-sanitizer over the device-resident partitioned BFS KATs (virtual
# ranks P = 1..4 and the s16 R-MAT cases): memcheck, racecheck, synccheck.
# Usage (GPU box): bash tools/sanitize_pdbfs.sh gpurun_out/sanitize_pd
set -u
OUT=${1:-gpurun_out/sanitize_pd}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
SMALL="tests/test_pdbfs_gpu.py::test_kat_virtual_ranks tests/test_pdbfs_gpu.py::test_push_only_virtual_ranks"
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout 1200 $CS --tool $tool $extra --kernel-name regex=k_pdbfs \
    --print-limit 50 --error-exitcode 99 --log-file "$OUT/$tool.log" \
    python -m pytest $SMALL -x -q -p no:cacheprovider > "$OUT/$tool.pytest.txt" 2>&1
  echo "$tool exit $?" | tee -a "$OUT/summary.txt"
  tail -3 "$OUT/$tool.log" >> "$OUT/summary.txt"
done
