set -x
python -m pytest tests/test_gpu_slab.py tests/test_gpu_paths.py -x -q -m gpu > gpurun_out/slab_tests.log 2>&1; echo slabtests=$?
tail -5 gpurun_out/slab_tests.log
python tools/run_configs.py C2 --steps 5 > gpurun_out/slab4_c2.jsonl 2> gpurun_out/slab4_c2.err
for v in b4 b6; do
  echo "== $v" >> gpurun_out/slab4_c2.jsonl
  TG_LIB_PATH=exp_variants/slab_$v/libtrigraph_b200.so python tools/run_configs.py C2 --steps 5 >> gpurun_out/slab4_c2.jsonl 2>> gpurun_out/slab4_c2.err
done
python tools/run_configs.py C5 --steps 3 > gpurun_out/slab4_c5.jsonl 2> gpurun_out/slab4_c5.err
python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo gputests=$?
tail -5 gpurun_out/gpu_tests.log
