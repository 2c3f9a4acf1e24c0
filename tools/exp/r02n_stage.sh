set -x
TG_LIB_PATH=exp_variants/stage/libtrigraph_b200.so python -m pytest tests/test_gpu_slab.py -x -q -m gpu > gpurun_out/r02n_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r02n_tests.log
for v in stage stage_b4; do
  echo "== $v" >> gpurun_out/r02n_c2.jsonl
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/run_configs.py C2 --steps 8 >> gpurun_out/r02n_c2.jsonl 2>> gpurun_out/r02n.err
  echo "== $v" >> gpurun_out/r02n_c5.jsonl
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/run_configs.py C5 --steps 4 >> gpurun_out/r02n_c5.jsonl 2>> gpurun_out/r02n.err
done
echo "== default" >> gpurun_out/r02n_c5.jsonl
python tools/run_configs.py C5 --steps 4 >> gpurun_out/r02n_c5.jsonl 2>> gpurun_out/r02n.err
