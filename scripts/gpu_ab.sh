# A/B of stage-kernel variants (scripts/variant_probe.py; bitwise against the first variant)
# usage: bash scripts/gpu_ab.sh TAG "c2 c5 c4" "auto brick_nb ..."
TAG=$1; CFGS=$2; VARS=$3
for c in $CFGS; do timeout 900 python scripts/variant_probe.py $c $VARS > gpurun_out/${TAG}_ab_$c.log 2>&1; done
echo finished
