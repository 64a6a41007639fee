# ncu --set full of the stage kernels (one launch each: the 3rd stage of the
# 4th RK3 step) for the brick configurations, plus the launch list of the
# headline bench command; every command runs once without ncu first
TAG=${1:-d}
for spec in c2:weno5 c4:weno5 c5:weno5 c2:weno5_fma; do
  cfg=${spec%%:*}; sch=${spec##*:}
  SCHEME=$sch timeout 600 python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_plain_${cfg}_$sch.log 2>&1 && \
  SCHEME=$sch timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 11 -c 1 \
      -o gpurun_out/${TAG}_prof_${cfg}_$sch python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_ncu_${cfg}_$sch.log 2>&1
done
timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/${TAG}_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_plain_bench_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
    python bench.py --config c4 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch_c4.log 2>&1
echo finished
