set -x
timeout 600 python bench.py > gpurun_out/z_bench.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/z_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/z_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/z_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/z_prof python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/z_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/z_prof_fma python bench.py --scheme weno5_fma --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/z_ncu_full_fma.log 2>&1
echo done
