mkdir -p gpurun_out/exp21
for k in 1 2 3; do
for v in _d3 _d2; do
  TS_LIB_PATH=paper_2604_00510_b200/lib/libtreeserve_b200$v.so timeout 120 python tools/graph_step_times.py >> gpurun_out/exp21/steps.txt 2>&1
done
done
