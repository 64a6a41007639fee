# full round check of the committed kernel: smoke, GPU parity suite, bench, launch list, ncu --set full
set -x
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/r_smoke.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r_plain.log 2>&1
timeout 600 python bench.py > gpurun_out/r_bench.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 --durations=15 > gpurun_out/r_pytest_gpu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/r_prof python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r_ncu_full.log 2>&1
echo done
