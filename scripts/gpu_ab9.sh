set -x
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > gpurun_out/r9_pytest.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/r9_bench.log 2>&1
HJ_STAGE_KERNEL=brick_u2 timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/r9_bench_u2.log 2>&1
timeout 300 python scripts/bench_configs.py c4 c5 > gpurun_out/r9_configs.log 2>&1
echo done
