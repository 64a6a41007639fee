cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v1_smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/v1_gputests.log 2>&1; echo "pytest rc $?" >> gpurun_out/v1_gputests.log
timeout 600 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/v1_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/v1_smoke.log
timeout 900 python bench.py > gpurun_out/v1_bench_c2.log 2>&1; echo "bench rc $?" >> gpurun_out/v1_bench_c2.log
