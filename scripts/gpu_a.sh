set -x
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/a_smoke.log 2>&1
bash scripts/gpu_multirank.sh
for cfg in c1 c2 c3 c4 c5; do timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/a_bench_$cfg.log 2>&1; done
echo finished
