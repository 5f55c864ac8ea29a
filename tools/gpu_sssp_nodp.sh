for i in 1 2; do
 echo -n "dp   "; python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-30
 echo -n "nodp "; GFX_SSSP_NODP=1 python tools/prof_run.py --prim sssp --delta 32 --scale 24 --runs 3 2>&1 | grep device_ms | cut -c1-30
done
python -c "import torch; p=torch.cuda.get_device_properties(0); print('persist max', getattr(p,'persisting_l2_cache_max_size',None), 'l2', p.L2_cache_size)"
