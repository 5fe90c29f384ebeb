#!/bin/bash
# On the GPU box: export the details and source pages of every .ncu-rep under $1
# (csv, the source page gzipped) and delete the reports, so that gpurun_out/
# stays under gpurun's copy-back limit.  tools/ncu_summary.py reads the exports.
for r in "$1"/*.ncu-rep; do
  [ -e "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i "$r" --page details --csv > "$b.details.csv" 2>/dev/null
  ncu -i "$r" --page source --csv --print-source=cuda,sass 2>/dev/null | gzip > "$b.source.csv.gz"
  rm -f "$r"
done
du -sh "$1"
