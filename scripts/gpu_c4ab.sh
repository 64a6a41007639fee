cd _ab/old && timeout 300 python scripts/bench_configs.py c4 c4 > ../../gpurun_out/l_c4_old.log 2>&1; cd ../..
timeout 300 python scripts/bench_configs.py c4 c4 > gpurun_out/l_c4_new.log 2>&1
timeout 600 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider -k "4d" > gpurun_out/l_pytest.log 2>&1
echo done
