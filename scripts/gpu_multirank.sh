# multi-rank slab path on one GPU (gloo-staged halos) + launch list
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/check_multirank.py --backend gloo > gpurun_out/multirank2.log 2>&1
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 3 scripts/check_multirank.py --backend gloo > gpurun_out/multirank3.log 2>&1
HJ_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_gloo.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
