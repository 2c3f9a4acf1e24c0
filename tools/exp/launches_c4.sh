# per-kernel launch list of one C4 step (orientation + count)
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_configs.py C4 --steps 1 > gpurun_out/x3_c4_launches.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_window -c 4 -o gpurun_out/x3_c4_window python tools/run_configs.py C4 --steps 1 > gpurun_out/x3_c4_full.log 2>&1
