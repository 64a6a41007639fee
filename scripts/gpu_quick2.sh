# quick kernel iteration: parity (golden + oracle under all kernel families), bench x2, ncu of the stage kernel
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_oracle.py tests/test_gpu_distributed.py -x -q -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline >> gpurun_out/q_bench.log 2>&1; done
timeout 600 python scripts/bench_configs.py c4 c5 > gpurun_out/q_configs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/q_prof python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/q_ncu.log 2>&1
echo done
