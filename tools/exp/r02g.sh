set -x
python -m pytest tests/test_gpu_comm.py tests/test_gpu_slab.py -x -q -m gpu > gpurun_out/comm_tests.log 2>&1; echo commtests=$?
tail -5 gpurun_out/comm_tests.log
for v in v3b5 curb5 v3b4 curb4 v3b5 curb5; do
  echo "== $v" >> gpurun_out/slab5_c2.jsonl
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/run_configs.py C2 --steps 8 >> gpurun_out/slab5_c2.jsonl 2>> gpurun_out/slab5_c2.err
done
for v in v3b5 curb5 v3b4 curb4; do
  echo "== $v" >> gpurun_out/slab5_c5.jsonl
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/run_configs.py C5 --steps 4 >> gpurun_out/slab5_c5.jsonl 2>> gpurun_out/slab5_c5.err
done
