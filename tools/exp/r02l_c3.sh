set -x
python tools/run_configs.py C3 --steps 3 > gpurun_out/r02l_c3.jsonl 2> gpurun_out/r02l_c3.err
cat gpurun_out/r02l_c3.jsonl
python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02l_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r02l_tests.log
python -m pytest tests/test_gpu_full.py -x -q -m gpu -k "C3 or c3 or config3" > gpurun_out/r02l_full3.log 2>&1; echo full=$?
tail -3 gpurun_out/r02l_full3.log
