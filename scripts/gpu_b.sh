set -x
nproc; free -g | head -2
timeout 600 python scripts/variant_probe.py c2 auto brick_noload > gpurun_out/b_var_c2.log 2>&1
timeout 600 python scripts/variant_probe.py c4 auto brick_noload > gpurun_out/b_var_c4.log 2>&1
timeout 600 python scripts/variant_probe.py c5 auto brick_noload > gpurun_out/b_var_c5.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=30 > gpurun_out/b_pytest.log 2>&1
echo finished
