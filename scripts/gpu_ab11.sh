timeout 1200 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_golden.py tests/test_gpu_distributed.py tests/test_gpu_batch.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider --timeout 900 > gpurun_out/r11_pytest.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r11_bench.log 2>&1
timeout 300 python scripts/bench_configs.py c4 c5 > gpurun_out/r11_c.log 2>&1
echo done
