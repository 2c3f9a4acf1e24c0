# slab layout probe + L2 fetch granularity on the real pass (C2, C5)
set -x
./tools/exp/slab_probe 1e8 2e7 > gpurun_out/slab_probe.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/slab_probe_ncu.csv ./tools/exp/slab_probe 1e8 2e7 > /dev/null 2>&1
python tools/exp/l2_fetch.py C2 3 > gpurun_out/l2_fetch_c2.jsonl 2> gpurun_out/l2_fetch_c2.err
python tools/exp/l2_fetch.py C5 3 > gpurun_out/l2_fetch_c5.jsonl 2> gpurun_out/l2_fetch_c5.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct
ncu --metrics $M --clock-control none -k regex:k_intersect_quad --csv --log-file gpurun_out/l2_fetch_c5_ncu.csv python tools/exp/l2_fetch.py C5 1 > gpurun_out/l2_fetch_c5_ncu.log 2>&1
echo done
