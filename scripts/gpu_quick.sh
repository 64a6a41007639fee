# quick: smoke + parity tests + bench + configs + ncu of the brick kernel
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_brick.log 2>&1
timeout 600 python scripts/bench_configs.py c1 c5 c4 > gpurun_out/configs.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/prof_brick6 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
