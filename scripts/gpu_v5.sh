# fused-schedule brick kernel: parity (all kernel families), bench, ncu of the stage kernel
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/v5_smoke.log 2>&1; echo smoke=$? >> gpurun_out/v5_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v5_pytest.log 2>&1
for v in brick brick; do
  HJ_STAGE_KERNEL=$v timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline >> gpurun_out/v5_bench.log 2>&1
done
timeout 600 python scripts/bench_configs.py c4 c5 > gpurun_out/v5_configs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/prof_v5 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_v5.log 2>&1
echo done
