timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_oracle.py tests/test_gpu_distributed.py tests/test_gpu_dd.py tests/test_gpu_cli.py -x -q -p no:cacheprovider > gpurun_out/i_pytest.log 2>&1
timeout 600 python scripts/variant_probe.py c4 auto > gpurun_out/i_var_c4.log 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/i_bench_c1.log 2>&1
echo finished
