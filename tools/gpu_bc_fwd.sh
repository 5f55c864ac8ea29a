timeout 1200 python -m pytest -q -x tests/test_analytics_gpu.py tests/test_parity_full_gpu.py tests/test_suite_gpu.py tests/test_operator_replay_gpu.py -k "bc or BC or suite" 2>&1 | tail -2
for r in 1 2 3; do
  echo "push $(GFX_BC_FWD=push python tools/bc_prof.py 22)"; echo "do   $(python tools/bc_prof.py 22)"
done
