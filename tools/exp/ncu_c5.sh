# full ncu captures of the C5 orientation and intersection kernels (one launch each)
ncu --set full --import-source on --clock-control none -k regex:"k_orient_tiles|k_intersect_quad" -c 2 -o gpurun_out/x10_c5 python tools/run_configs.py C5 --steps 1 > gpurun_out/x10.log 2>&1
