#!/bin/bash
# All ncu evidence of one round in one GPU call (run under gpurun; outputs in gpurun_out/).
# Summaries for profiles/ are made here afterwards with tools/ncu_summary.py.
set -x
O=gpurun_out/prof
mkdir -p $O
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launch_c2_full.csv python tools/prof_driver.py full
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launch_c2_exits_off.csv python tools/prof_driver.py exits_off
$NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:'k_wave|k_heavy' --csv --log-file $O/dram_c2_full.csv python tools/prof_driver.py full
$NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:'k_wave|k_heavy' --csv --log-file $O/dram_c2_exits_off.csv python tools/prof_driver.py exits_off
$NCU --set full --import-source on -k regex:k_heavy --launch-skip 3 --launch-count 1 -f -o $O/heavy_tail python tools/prof_driver.py full
$NCU --set full --import-source on -k regex:k_wave --launch-count 1 -f -o $O/wave_first python tools/prof_driver.py full
$NCU --set full --import-source on -k regex:k_wave --launch-skip 60 --launch-count 1 -f -o $O/wave_exits_off python tools/prof_driver.py exits_off
$NCU --set full --import-source on -k regex:k_beam --launch-skip 1 --launch-count 1 -f -o $O/beam python tools/beam_driver.py
$NCU --set full -k regex:'k_sort_tile|k_targets_out|k_scores' --launch-skip 12 --launch-count 3 -f -o $O/ct python tools/ct_prof.py
# the graph loop's scheduler pass (ncu cannot profile kernels of a conditional graph: host-driven stepping)
TS_NO_GRAPH=1 $NCU --set full --import-source on -k regex:k_sched --launch-skip 2 --launch-count 1 -f -o $O/ksched python bench.py --steps 1 --warmup 3 > $O/ksched_bench.log 2>&1
# per-phase timers of the graph loop (the -DTS_SCHED_PROF build)
[ -f paper_2604_00510_b200/lib/libtreeserve_b200_sprof.so ] && { python tools/sched_prof.py > $O/sched_prof.txt 2>&1; python tools/sched_prof.py exits_off >> $O/sched_prof.txt 2>&1; }
ls -la $O
