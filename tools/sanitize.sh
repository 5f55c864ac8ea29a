#!/bin/bash
# compute-sanitizer over the GPU KAT suite (s <= 16): memcheck, racecheck,
# synccheck, initcheck on every libgfx kernel the small tests launch.
# Usage (GPU box): bash tools/sanitize.sh gpurun_out/sanitize
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
SMALL="tests/test_bfs_gpu.py::test_kat_bfs_all_modes tests/test_bfs_gpu.py::test_reference_kats \
tests/test_bfs_gpu.py::test_s16_golden tests/test_sssp_gpu.py::test_kat_sssp \
tests/test_sssp_gpu.py::test_s16_golden tests/test_analytics_gpu.py::test_kat_all \
tests/test_operators_gpu.py tests/test_operator_replay_gpu.py \
tests/test_dist_gpu.py::test_kat_partitioned tests/test_dist_sssp_gpu.py::test_kat_partitioned_sssp"
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout 1500 $CS --tool $tool $extra --kernel-name regex=_ZN3gfx \
    --print-limit 50 --error-exitcode 99 --log-file "$OUT/$tool.log" \
    python -m pytest $SMALL -x -q -p no:cacheprovider > "$OUT/$tool.pytest.txt" 2>&1
  echo "$tool exit $?" | tee -a "$OUT/summary.txt"
  tail -3 "$OUT/$tool.log" >> "$OUT/summary.txt"
done
