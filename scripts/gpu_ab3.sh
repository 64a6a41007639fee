# A/B of the WENO5 walk unroll (brick vs brick_u4 vs brick1) + parity + ncu of the winner candidate
for v in brick brick_u4 brick1; do
  HJ_STAGE_KERNEL=$v timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done
HJ_STAGE_KERNEL=brick_u4 timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_oracle.py -q -p no:cacheprovider -x > gpurun_out/pytest_u4.log 2>&1
v=brick_u4
HJ_STAGE_KERNEL=$v timeout 300 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain_$v.log 2>&1 && \
HJ_STAGE_KERNEL=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/prof_$v python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$v.log 2>&1
echo done
