timeout 600 python -m pytest -q -x tests/test_pack_gpu.py 2>&1 | tail -3
GFX_REBUILD=sort timeout 600 python -m pytest -q -x tests/test_pack_gpu.py -k upper 2>&1 | tail -2
timeout 300 python tools/e2e_parts.py > gpurun_out/e2e_parts.txt 2>&1
GFX_REBUILD=sort timeout 300 python tools/e2e_parts.py > gpurun_out/e2e_parts_sort.txt 2>&1
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/e2e_bench.json 2> gpurun_out/e2e_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/e2e_bench.json').read().strip().splitlines()[-1]); e=d['e2e']
print(d['value'], e['value'], e['ms_per_step'], e['h2d_bytes_per_step'], e['batches_ms_per_step'], e['packed_full_csr'])"
tail -4 gpurun_out/e2e_parts.txt; tail -3 gpurun_out/e2e_parts_sort.txt; tail -3 gpurun_out/e2e_bench.err
