# multi-rank slab paths on a one-GPU lease:
#  * NCCL data plane (hj_dd) as a one-rank periodic ring (tests/test_gpu_dd.py)
#  * torchrun ranks sharing the GPU over gloo-staged halos (check_multirank.py,
#    bench.py with HJ_SLAB_COMM=torch) -- no kernel waits on another rank
timeout 900 python -m pytest tests/test_gpu_dd.py tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/mr_pytest.log 2>&1
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/check_multirank.py --backend gloo > gpurun_out/mr_check2.log 2>&1
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 3 scripts/check_multirank.py --backend gloo --planes 40 --steps 1 > gpurun_out/mr_check3.log 2>&1
for cfg in c2 c3 c4 c5; do
  HJ_SLAB_COMM=torch timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config $cfg --size 40 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/mr_bench_$cfg.log 2>&1
done
echo done
