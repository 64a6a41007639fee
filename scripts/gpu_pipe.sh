set -x
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_oracle.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/q_pytest.log 2>&1
timeout 300 python bench.py --e2e-steps 5 --no-cpu-baseline --steps 10 > gpurun_out/q_bench.log 2>&1
echo done
