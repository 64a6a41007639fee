# brick load rewrite: parity (brick tests) + both benches + ncu of both kernels
set -x
timeout 900 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_weno_fma.py tests/test_gpu_distributed.py tests/test_gpu_batch.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/i_pytest.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/i_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/i_prof_exact python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/i_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/i_prof_fma python bench.py --scheme weno5_fma --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/i_ncu2.log 2>&1
echo done
