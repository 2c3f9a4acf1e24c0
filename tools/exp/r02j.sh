set -x
python -X faulthandler bench.py --config C1 --no-cpu --force-comm --steps 3 > gpurun_out/r02j_c1_comm1.json 2> gpurun_out/r02j_c1_comm1.log; echo rc=$?
tail -5 gpurun_out/r02j_c1_comm1.log
python -X faulthandler bench.py --config C2 --no-cpu --force-comm --steps 5 > gpurun_out/r02j_c2_comm1.json 2> gpurun_out/r02j_c2_comm1.log; echo rc=$?
tail -30 gpurun_out/r02j_c2_comm1.log
python tools/run_configs.py C5 --steps 4 > gpurun_out/r02j_orient_c5.jsonl 2> gpurun_out/r02j_orient_c5.err
for v in tie_b4 tie_b4u6; do
  echo "== $v" >> gpurun_out/r02j_orient_c5.jsonl
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/run_configs.py C5 --steps 4 >> gpurun_out/r02j_orient_c5.jsonl 2>> gpurun_out/r02j_orient_c5.err
done
python -m pytest tests/test_gpu_paths.py tests/test_gpu_slab.py -x -q -m gpu > gpurun_out/r02j_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r02j_tests.log
