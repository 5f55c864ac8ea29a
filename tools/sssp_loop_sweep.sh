# SSSP s24 device-resident vs host-driven loop over delta
for m in device host; do echo "== $m"; GFX_SSSP_LOOP=$m python tools/sssp_delta_sweep.py 2>&1 | tail -8; done
