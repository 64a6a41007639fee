# A/B of two builds of libhjb200 on one box: the in-tree build against
# _ab/libhjb200_<REV>.so (HJ_LIB_PATH), alternating, per BASELINE config
# (scripts/variant_probe.py "auto": 20 RK3 steps after 3, CUDA events).
TAG=${1:-abb}; REV=${2:?rev}
for cfg in c2 c5 c4; do
  for k in 1 2; do
    HJ_LIB_PATH=$PWD/_ab/libhjb200_$REV.so timeout 600 python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_${cfg}_${REV}_$k.log 2>&1
    timeout 600 python scripts/variant_probe.py $cfg auto > gpurun_out/${TAG}_${cfg}_head_$k.log 2>&1
  done
done
echo done
