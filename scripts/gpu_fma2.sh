set -x
timeout 900 python -m pytest tests/test_gpu_weno_fma.py -q -p no:cacheprovider --timeout 600 --durations=5 > gpurun_out/g_pytest.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/g_bench.log 2>&1
HJ_STAGE_KERNEL=brick_u2 timeout 300 python bench.py --scheme weno5_fma --e2e-steps 0 --no-cpu-baseline > gpurun_out/g_bench_u2.log 2>&1
echo done
