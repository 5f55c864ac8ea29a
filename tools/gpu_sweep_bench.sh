# bench-mode timing of variant builds: bash tools/gpu_sweep_bench.sh base v1 v2 ...
# (paper_1701_01170_b200/libgfx_<name>.so each), two alternations
for round in 1 2; do
for v in "$@"; do
  GFX_LIB_PATH=$PWD/paper_1701_01170_b200/libgfx_$v.so python bench.py --no-extras --no-e2e --no-cpu-baseline > gpurun_out/sweep_$v.json 2> gpurun_out/sweep_$v.err
  echo -n "$v rc=$? "; python -c "import sys,json; d=json.loads(open('gpurun_out/sweep_$v.json').read()); print(d['value'], d['ms_per_step'], [round(l['ms']*1000,1) for l in d['roofline']['levels']])" 2>/dev/null || tail -2 gpurun_out/sweep_$v.err
done; done
