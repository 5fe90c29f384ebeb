mkdir -p gpurun_out/exp20
for k in 1 2 3; do
for v in _sel32 _sel0; do
  FLUSH=1 TS_LIB_PATH=paper_2604_00510_b200/lib/libtreeserve_b200$v.so timeout 120 python tools/graph_step_times.py >> gpurun_out/exp20/steps.txt 2>&1
  TS_LIB_PATH=paper_2604_00510_b200/lib/libtreeserve_b200$v.so timeout 120 python tools/graph_step_times.py >> gpurun_out/exp20/steps.txt 2>&1
done
done
