timeout 1200 python -m pytest -q -x tests/test_bfs_gpu.py tests/test_analytics_gpu.py tests/test_headline*.py tests/test_parity_full_gpu.py::test_bfs_s27_vs_host_c_oracle tests/test_operators_gpu.py 2>&1 | tail -2
bash tools/gpu_ab_multi.sh 6 base pinit 2>&1 | tail -4
