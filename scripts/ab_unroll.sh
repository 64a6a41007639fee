# A/B of the per-axis walk pipeline's loop-unroll variants on the BASELINE
# grids (scripts/variant_probe.py: 20 RK3 steps after 3, CUDA events; each
# variant checked bitwise against "auto" after the same 23 steps), then the
# GPU parity tests of the per-axis kernel family.
TAG=${1:-abu}
for cfg in c2 c5 c4; do
  timeout 900 python scripts/variant_probe.py $cfg auto axes_s32 auto > gpurun_out/${TAG}_ab_$cfg.log 2>&1
done
[ -n "$SKIP_TESTS" ] || { timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_tests.log; }
echo done
