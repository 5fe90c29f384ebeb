#!/bin/bash
# Round-2 ncu evidence in one GPU call (run under gpurun; outputs in gpurun_out/prof2/).
# Summaries for profiles/ are made afterwards with tools/ncu_summary.py.
set -x
O=gpurun_out/prof2
mkdir -p $O
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launch_c2_full.csv python tools/prof_driver.py full
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launch_c2_exits_off.csv python tools/prof_driver.py exits_off
$NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:'k_wave|k_heavy' --csv --log-file $O/dram_c2_full.csv python tools/prof_driver.py full
$NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:'k_wave|k_heavy' --csv --log-file $O/dram_c2_exits_off.csv python tools/prof_driver.py exits_off
$NCU --set full --import-source on -k regex:k_heavy --launch-skip 3 --launch-count 1 -f -o $O/heavy_tail python tools/prof_driver.py full
$NCU --set full --import-source on -k regex:k_wave --launch-count 1 -f -o $O/wave_first python tools/prof_driver.py full
$NCU --set full --import-source on -k regex:k_wave --launch-skip 60 --launch-count 1 -f -o $O/wave_exits_off python tools/prof_driver.py exits_off
TS_NO_GRAPH=1 $NCU --set full --import-source on -k regex:k_sched --launch-skip 2 --launch-count 1 -f -o $O/ksched python bench.py --steps 1 --warmup 3 > $O/ksched_bench.log 2>&1
# the sharded loop's fused scheduler step (one rank, config-3 shape, the graph's kernels are visible to ncu
# only outside a conditional graph: the driver below runs ts_run_sharded; ncu profiles its graph kernels)
$NCU --set full --import-source on -k regex:k_px_step --launch-skip 5 --launch-count 1 -f -o $O/px_step python tools/peer_overhead.py 1 4096 > $O/px_step.log 2>&1
ls -la $O
