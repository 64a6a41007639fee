python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1
for v in brick brick1; do
  HJ_STAGE_KERNEL=$v timeout 300 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done
HJ_STAGE_KERNEL=brick1 timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_oracle.py -q -p no:cacheprovider -x > gpurun_out/pytest_brick1.log 2>&1
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 3 scripts/check_multirank.py --backend gloo --planes 301 --steps 1 > gpurun_out/multirank3.log 2>&1
for v in brick brick1; do
HJ_STAGE_KERNEL=$v timeout 300 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain_$v.log 2>&1 && \
HJ_STAGE_KERNEL=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/prof_$v python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$v.log 2>&1
done
echo done
