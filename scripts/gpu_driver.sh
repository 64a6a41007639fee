# what the driver runs at round end (1 GPU), plus the launch list for profiles/
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
