set -x
python tools/run_configs.py C3 --steps 3 > gpurun_out/r02r_c3.jsonl 2> gpurun_out/r02r_c3.err
for v in cph128 cph512; do
  echo "== $v" >> gpurun_out/r02r_c3.jsonl
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/run_configs.py C3 --steps 3 >> gpurun_out/r02r_c3.jsonl 2>> gpurun_out/r02r_c3.err
done
cat gpurun_out/r02r_c3.jsonl | cut -c1-60,230-420
python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_orders.py -x -q -m gpu > gpurun_out/r02r_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r02r_tests.log
python -m pytest tests/test_gpu_full.py -x -q -m gpu > gpurun_out/r02r_full.log 2>&1; echo full=$?
tail -3 gpurun_out/r02r_full.log
