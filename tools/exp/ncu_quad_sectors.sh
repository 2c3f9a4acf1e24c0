set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
python tools/run_configs.py C2 --steps 2 > gpurun_out/x1_c2.log 2>&1
ncu --metrics $M --clock-control none -k regex:k_intersect_quad -c 2 --csv python tools/run_configs.py C2 --steps 1 > gpurun_out/x1_ncu_base.csv 2>&1
TG_LIB_PATH=$PWD/exp_variants/ldg/libtrigraph_b200.so ncu --metrics $M --clock-control none -k regex:k_intersect_quad -c 2 --csv python tools/run_configs.py C2 --steps 1 > gpurun_out/x1_ncu_ldg.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_intersect_quad -c 1 -o gpurun_out/x1_quad_c2 python tools/run_configs.py C2 --steps 1 > gpurun_out/x1_ncu_full.log 2>&1
ls -la gpurun_out
