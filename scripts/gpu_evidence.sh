# Round evidence in one gpurun call (writes gpurun_out/${TAG}_*):
#  smoke; ncu --set full of the stage kernels + FP64 stamps and DRAM traffic
#  (profiles/fp64_ops.json, traffic.json, copied to gpurun_out/); the bench
#  line of every config; the reference arm of every config; launch lists.
TAG=${1:-ev}
[ -n "$SKIP_TESTS" ] || timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_gputests.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_gputests.log
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
rm -f profiles/fp64_ops.json profiles/traffic.json
# one stage's kernels (the RK3 third stage of the 4th step): the per-axis walk
# pipeline for WENO5 (dim kernels per stage), the brick kernel for weno5_fma
for spec in c2:weno5:27270901:k_axis:3 c4:weno5:214358881:k_axis:4 c5:weno5:8242408:k_axis:3 \
            c2:weno5_fma:27270901:k_stage_brick:1; do
  IFS=: read cfg sch nodes kre nk <<< "$spec"
  SCHEME=$sch timeout 600 python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_plain_${cfg}_$sch.log 2>&1 && \
  SCHEME=$sch timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $((11 * nk)) -c $nk \
      -o gpurun_out/${TAG}_prof_${cfg}_$sch python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_ncu_${cfg}_$sch.log 2>&1 && \
  python scripts/ncu_summary.py gpurun_out/${TAG}_prof_${cfg}_$sch.ncu-rep $nodes --stamp ${cfg}_$sch --traffic ${cfg}_${sch}_1 \
      > gpurun_out/${TAG}_ncu_${cfg}_$sch.json 2>&1
  # per-instruction source page (scripts/sass_regions.py), then drop the report
  # (gpurun copies back at most 64 MiB of gpurun_out/)
  ncu -i gpurun_out/${TAG}_prof_${cfg}_$sch.ncu-rep --page source --csv --print-source sass \
      > gpurun_out/${TAG}_src_${cfg}_$sch.csv 2>/dev/null && gzip -f gpurun_out/${TAG}_src_${cfg}_$sch.csv
  rm -f gpurun_out/${TAG}_prof_${cfg}_$sch.ncu-rep
done
# C1: the persistent tile kernel (one launch = one interval of 158 ENO2/RK2 stages of 93636 nodes)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_persist -s 2 -c 1 \
    -o gpurun_out/${TAG}_prof_c1_eno2 python scripts/c1_persist_probe.py auto > gpurun_out/${TAG}_ncu_c1_eno2.log 2>&1 && \
python scripts/ncu_summary.py gpurun_out/${TAG}_prof_c1_eno2.ncu-rep 14794488 > gpurun_out/${TAG}_ncu_c1_eno2.json 2>&1
rm -f gpurun_out/${TAG}_prof_c1_eno2.ncu-rep
cp profiles/fp64_ops.json gpurun_out/${TAG}_fp64_ops.json; cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
for cfg in c2 c1 c3 c4 c5; do timeout 900 python bench.py --config $cfg > gpurun_out/${TAG}_bench_$cfg.log 2>&1; done
for cfg in c2 c1 c3 c4 c5; do timeout 900 python bench.py --impl reference --config $cfg > gpurun_out/${TAG}_bench_ref_$cfg.log 2>&1; done
timeout 300 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/${TAG}_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-tolerance-mode > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo finished
HJ_LIB=check timeout 900 python scripts/bounds_check.py > gpurun_out/${TAG}_bounds.txt 2>&1; echo "rc $?" >> gpurun_out/${TAG}_bounds.txt
