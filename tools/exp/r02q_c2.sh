set -x
B="python bench.py --config C2 --no-cpu --steps 2 --warmup 3 --e2e-steps 1 --e2e-warmup 0"
$B > gpurun_out/r02q_plain.json 2> gpurun_out/r02q_plain.log
ncu --set full --import-source on --clock-control none -k regex:"k_intersect_slab|k_orient_tiles" -s 6 -c 2 -o gpurun_out/r02q_c2_step $B > gpurun_out/r02q_ncu.log 2>&1
