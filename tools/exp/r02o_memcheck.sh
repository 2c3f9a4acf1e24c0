set -x
python tools/exp/memcheck_slab.py > gpurun_out/r02o_plain.log 2>&1; echo plain=$?
tail -5 gpurun_out/r02o_plain.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/exp/memcheck_slab.py > gpurun_out/r02o_memcheck.log 2>&1; echo memcheck=$?
tail -15 gpurun_out/r02o_memcheck.log
