# perfect-hash slab kernel: correctness, C2 / C5 timing, variants, ncu of the C5 step
set -x
python -m pytest tests/test_gpu_slab.py -x -q -m gpu > gpurun_out/slab_tests.log 2>&1; echo slabtests=$?
tail -5 gpurun_out/slab_tests.log
python tools/run_configs.py C2 --steps 5 > gpurun_out/slab3_c2.jsonl 2> gpurun_out/slab3_c2.err
for v in b6u6 b4u6 b5u5 b5u7; do
  echo "== $v" >> gpurun_out/slab3_c2.jsonl
  TG_LIB_PATH=exp_variants/slab_$v/libtrigraph_b200.so python tools/run_configs.py C2 --steps 5 >> gpurun_out/slab3_c2.jsonl 2>> gpurun_out/slab3_c2.err
done
python tools/run_configs.py C5 --steps 3 > gpurun_out/slab3_c5.jsonl 2> gpurun_out/slab3_c5.err
ncu --set full --import-source on --clock-control none -k regex:"k_intersect_slab|k_orient_tiles" -s 4 -c 2 -o gpurun_out/r02e_c5 python tools/run_configs.py C5 --steps 1 > gpurun_out/ncu_c5.log 2>&1
echo done
