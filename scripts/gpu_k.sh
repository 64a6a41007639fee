HJ_LIB=check timeout 1200 python scripts/bounds_check.py > gpurun_out/k_bounds.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_plugins.py tests/test_gpu_golden.py tests/test_gpu_dd.py tests/test_gpu_cli.py tests/test_gpu_baseline_sizes.py -x -q -p no:cacheprovider -k "not 101 and not c3_size and not c5_batch" > gpurun_out/k_pytest.log 2>&1
echo finished
