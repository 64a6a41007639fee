for k in brick brick_u2 brick1; do
HJ_STAGE_KERNEL=$k timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode --steps 20 > gpurun_out/k_bench_$k.log 2>&1
done
echo done
