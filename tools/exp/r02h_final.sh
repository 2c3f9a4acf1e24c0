# round-2 measurement set: tests, the C5 bench (both arms), launch list, full capture, other configs, projection
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/r02h_gputest.log 2>&1; echo gputests=$?
tail -3 gpurun_out/r02h_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo smoke=$?
python bench.py --impl reference > gpurun_out/r02h_bench_reference.json 2> gpurun_out/r02h_bench_reference.log; echo ref=$?
python bench.py > gpurun_out/r02h_bench_c5.json 2> gpurun_out/r02h_bench_c5.log; echo bench=$?
B="python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 --e2e-warmup 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_c5.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_intersect_slab|k_orient_tiles" -s 8 -c 2 -o gpurun_out/r02h_c5_step $B > gpurun_out/ncu_full.log 2>&1
python bench.py --config C2 --no-cpu > gpurun_out/r02h_bench_c2.json 2> gpurun_out/r02h_bench_c2.log
python tools/run_configs.py C3 C4 --steps 3 > gpurun_out/r02h_c3c4.jsonl 2> gpurun_out/r02h_c3c4.err
python tools/scaling_projection.py C2 C5 > gpurun_out/r02h_scaling.jsonl 2> gpurun_out/r02h_scaling.err
echo done
