set -x
timeout 900 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_weno_fma.py tests/test_gpu_distributed.py tests/test_gpu_batch.py tests/test_gpu_golden.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/j_pytest.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/j_bench.log 2>&1
HJ_STAGE_KERNEL=brick_u2 timeout 300 python bench.py --scheme weno5_fma --e2e-steps 0 --no-cpu-baseline > gpurun_out/j_bench_u4.log 2>&1
echo done
