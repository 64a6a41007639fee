# Final bench lines (no ncu): every config, both arms, into gpurun_out/${TAG}_*
TAG=${1:-fin}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gputests.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_gputests.log
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
for cfg in c2 c1 c3 c4 c5; do timeout 900 python bench.py --config $cfg > gpurun_out/${TAG}_bench_$cfg.log 2>&1; done
echo finished
