# ncu --set full of one RK3 stage of the per-axis pipeline at C2 (301^3) and
# C4 (121^4), per-kernel summary + per-instruction source page (gzip)
TAG=${1:-nc}
for spec in c2:27270901:3 c4:214358881:4; do
  IFS=: read cfg nodes nk <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_axis -s $((11 * nk)) -c $nk \
      -o gpurun_out/${TAG}_prof_$cfg python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_ncu_$cfg.log 2>&1 && \
  python scripts/ncu_summary.py gpurun_out/${TAG}_prof_$cfg.ncu-rep $nodes > gpurun_out/${TAG}_ncu_$cfg.json 2>&1
  ncu -i gpurun_out/${TAG}_prof_$cfg.ncu-rep --page source --csv --print-source sass \
      > gpurun_out/${TAG}_src_$cfg.csv 2>/dev/null && gzip -f gpurun_out/${TAG}_src_$cfg.csv
  rm -f gpurun_out/${TAG}_prof_$cfg.ncu-rep
done
echo done
