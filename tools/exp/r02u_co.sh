set -x
for c in C2 C5; do
python tools/exp/co_run.py $c >> gpurun_out/r02u_co.jsonl 2>> gpurun_out/r02u_co.err
for v in co22 co23 co32; do
  TG_LIB_PATH=exp_variants/$v/libtrigraph_b200.so python tools/exp/co_run.py $c >> gpurun_out/r02u_co.jsonl 2>> gpurun_out/r02u_co.err
done
done
cat gpurun_out/r02u_co.jsonl
