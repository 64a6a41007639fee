# tolerance-mode WENO5: parity vs oracle, bench A/B, ncu of the fma brick kernel
set -x
timeout 900 python -m pytest tests/test_gpu_weno_fma.py -q -p no:cacheprovider --timeout 600 --durations=10 > gpurun_out/f_pytest.log 2>&1
timeout 300 python bench.py --scheme weno5_fma --e2e-steps 2 --no-cpu-baseline > gpurun_out/f_bench_fma.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/f_bench_exact.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/f_prof python bench.py --scheme weno5_fma --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/f_ncu_full.log 2>&1
echo done
