#!/bin/bash
# A/B of heavy-CTA shapes: headline batch time (graph loop) and per-wave times.
for L in libtreeserve_b200.so libtreeserve_b200_h5_3.so libtreeserve_b200_h6_3.so; do
  echo "== $L"
  TS_LIB_PATH=paper_2604_00510_b200/lib/$L python tools/graph_step_times.py 2>&1 | head -1
  TS_LIB_PATH=paper_2604_00510_b200/lib/$L python tools/wave_targets.py 2>&1 | cut -c1-60
  TS_LIB_PATH=paper_2604_00510_b200/lib/$L python tools/wave_occupancy.py 2>&1 | head -2
done
