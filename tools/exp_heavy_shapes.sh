mkdir -p gpurun_out/exp1
for v in "" _w6b3 _w5b3 _w8b3 _w6r112; do
  for k in 1 2; do
  TS_LIB_PATH=paper_2604_00510_b200/lib/libtreeserve_b200$v.so timeout 120 python tools/graph_step_times.py >> gpurun_out/exp1/steps.txt 2>&1
  done
done
