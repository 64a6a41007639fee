timeout 300 python scripts/bench_configs.py c4 c5 > gpurun_out/r10_c_u1.log 2>&1
HJ_STAGE_KERNEL=brick_u2 timeout 300 python scripts/bench_configs.py c4 c5 > gpurun_out/r10_c_u2.log 2>&1
echo done
