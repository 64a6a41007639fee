# A/B: walk unroll 1 (brick) vs 2 (brick_u4 slot), plus ncu of the unroll-2 kernel
for v in brick brick_u4 brick brick_u4; do
  HJ_STAGE_KERNEL=$v timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline >> gpurun_out/ab4_$v.log 2>&1
done
v=brick_u4
HJ_STAGE_KERNEL=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/prof_u2 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_u2.log 2>&1
echo done
