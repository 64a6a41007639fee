# ncu --set full of the stage kernels (one launch each: the 3rd stage of a
# warm RK3 step) for the three brick configurations; plain runs first
TAG=${1:-d}
for cfg in c2 c4 c5; do
  timeout 600 python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_plain_$cfg.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 11 -c 1 \
      -o gpurun_out/${TAG}_prof_$cfg python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_ncu_$cfg.log 2>&1
done
echo finished
