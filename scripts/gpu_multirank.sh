# multi-rank slab path on one GPU (gloo-staged halos) + memcheck of the slab kernels
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/check_multirank.py --backend gloo > gpurun_out/multirank2.log 2>&1
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 3 scripts/check_multirank.py --backend gloo --n 301 --steps 1 > gpurun_out/multirank3.log 2>&1
HJ_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_gloo.log 2>&1
timeout 600 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_batch.py -q -p no:cacheprovider > gpurun_out/pytest_dist.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_distributed.py -q -p no:cacheprovider -k "weno5-2 or ring" > gpurun_out/memcheck.log 2>&1
echo done
