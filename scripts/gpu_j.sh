timeout 300 python scripts/variant_probe.py c4 auto > gpurun_out/j_plain_c4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/j_launches_c4.csv python scripts/variant_probe.py c4 auto > gpurun_out/j_ncu_c4.log 2>&1
timeout 300 python bench.py --config c1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/j_plain_c1.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 40 --csv --log-file gpurun_out/j_launches_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/j_ncu_c1.log 2>&1
echo finished
