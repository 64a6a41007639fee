# round evidence for the committed kernels: default bench line, reference arm,
# secondary configs, launch list (cold, serialised) and ncu --set full captures
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/p_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/p_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/p_bench_ref.log 2>&1
timeout 900 python scripts/bench_configs.py c1 c4 c5 c2s c4:weno5_fma c5:weno5_fma c2s:weno5_fma > gpurun_out/p_configs.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/p_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/p_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/p_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/p_prof python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/p_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 2 -c 1 -o gpurun_out/p_prof_fma python bench.py --scheme weno5_fma --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/p_ncu_full_fma.log 2>&1
echo done
