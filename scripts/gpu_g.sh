for cfg in c2 c4 c5; do timeout 600 python scripts/variant_probe.py $cfg auto brick_nopf > gpurun_out/g_var_$cfg.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_oracle.py -x -q -p no:cacheprovider > gpurun_out/g_pytest.log 2>&1
echo finished
