# C5 headline: reference arm, launch list and a full capture of the dominant kernel
set -x
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo ref=$?
B="python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 --e2e-warmup 0"
$B > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_intersect_quad|k_orient_tiles" -s 6 -c 2 -o gpurun_out/c5_step $B > gpurun_out/ncu_full.log 2>&1
echo done
