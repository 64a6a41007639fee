timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > gpurun_out/v_pytest.log 2>&1
timeout 300 python bench.py --e2e-steps 3 --no-cpu-baseline > gpurun_out/v_bench.log 2>&1
echo done
