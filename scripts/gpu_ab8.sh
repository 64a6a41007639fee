set -x
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > gpurun_out/o_pytest.log 2>&1
timeout 300 python scripts/bench_configs.py c4 c5 c4:weno5_fma > gpurun_out/o_configs.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/o_bench.log 2>&1
echo done
