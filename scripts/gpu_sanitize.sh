set -x
timeout 300 python scripts/sanitize_probe.py > gpurun_out/s_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python scripts/sanitize_probe.py > gpurun_out/s_racecheck.log 2>&1
echo rc=$?
