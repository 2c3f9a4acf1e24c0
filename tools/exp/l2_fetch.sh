# cudaLimitMaxL2FetchGranularity sweep on the intersection pass (C2, C5)
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
for f in 0 32 64 128; do
  echo "== fetch $f"
  TG_L2_FETCH=$f python tools/run_configs.py C2 --steps 3 2>&1 | grep -E "^\{|granularity"
done
TG_L2_FETCH=32 ncu --metrics $M --clock-control none -k regex:k_intersect_quad -c 1 --csv python tools/run_configs.py C2 --steps 1 > gpurun_out/x2_ncu_f32.csv 2>&1
TG_L2_FETCH=0 ncu --metrics $M --clock-control none -k regex:k_intersect_quad -c 1 --csv python tools/run_configs.py C2 --steps 1 > gpurun_out/x2_ncu_f0.csv 2>&1
for f in 32 0; do
  echo "== C5 fetch $f"
  TG_L2_FETCH=$f python tools/run_configs.py C5 --steps 3 2>&1 | grep -E "^\{|granularity"
done
