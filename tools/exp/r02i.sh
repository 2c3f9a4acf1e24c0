set -x
python -m pytest tests/test_gpu_comm.py tests/test_gpu_distributed.py tests/test_gpu_cpp.py -x -q -m gpu > gpurun_out/r02i_comm_tests.log 2>&1; echo commtests=$?
tail -5 gpurun_out/r02i_comm_tests.log
for v in ou2 ou6 ou8 ob6 ob4u8; do
  echo "== $v" >> gpurun_out/r02i_orient_c5.jsonl
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/run_configs.py C5 --steps 4 >> gpurun_out/r02i_orient_c5.jsonl 2>> gpurun_out/r02i_orient_c5.err
done
python tools/scaling_projection.py C5 > gpurun_out/r02i_scaling.jsonl 2> gpurun_out/r02i_scaling.err
python bench.py --config C2 --no-cpu --force-comm --steps 10 > gpurun_out/r02i_bench_c2_comm1.json 2> gpurun_out/r02i_bench_c2_comm1.log
