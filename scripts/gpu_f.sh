for cfg in c2 c4 c5; do timeout 600 python scripts/variant_probe.py $cfg auto brick_u2 brick_nopf auto > gpurun_out/f_var_$cfg.log 2>&1; done
echo finished
