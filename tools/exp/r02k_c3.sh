set -x
python tools/run_configs.py C3 --steps 2 > gpurun_out/r02k_c3.jsonl 2> gpurun_out/r02k_c3.err
ncu --set full --import-source on --clock-control none -k regex:"k_intersect_ctab|k_intersect_ctaq|k_intersect_groupq" -s 6 -c 3 -o gpurun_out/r02k_c3 python tools/run_configs.py C3 --steps 1 > gpurun_out/r02k_ncu.log 2>&1
