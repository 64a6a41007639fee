set -x
for cfg in c2 c4 c5; do timeout 600 python scripts/variant_probe.py $cfg auto > gpurun_out/e_var_$cfg.log 2>&1; done
HJ_REFERENCE_SUITE=1 timeout 1800 python -m pytest tests/reference_suite -m gpu -q -p no:cacheprovider -rs > gpurun_out/e_reference_suite.log 2>&1
echo finished
