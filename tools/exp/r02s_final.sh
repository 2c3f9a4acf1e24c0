# final check of the round: tests, smoke, both bench arms
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/r02s_gputest.log 2>&1; echo gputests=$?
tail -3 gpurun_out/r02s_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/r02s_smoke.log
python bench.py --impl reference > gpurun_out/r02s_bench_reference.json 2> gpurun_out/r02s_bench_reference.log; echo ref=$?
python bench.py > gpurun_out/r02s_bench_c5.json 2> gpurun_out/r02s_bench_c5.log; echo bench=$?
python tools/run_configs.py C3 C4 --steps 3 > gpurun_out/r02s_c3c4.jsonl 2> gpurun_out/r02s_c3c4.err
