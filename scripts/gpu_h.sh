timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_oracle.py tests/test_gpu_distributed.py tests/test_gpu_dd.py tests/test_gpu_batch.py tests/test_gpu_weno_fma.py -x -q -p no:cacheprovider > gpurun_out/h_pytest.log 2>&1
for cfg in c2 c4 c5; do timeout 600 python scripts/variant_probe.py $cfg auto > gpurun_out/h_var_$cfg.log 2>&1; done
echo finished
