# A/B of the stage kernels + correctness + profile, one GPU call
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1
for v in generic brick; do
  HJ_STAGE_KERNEL=$v timeout 300 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/prof_brick5 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 600 python scripts/bench_configs.py c1 c5 c2s > gpurun_out/configs.log 2>&1
echo done
