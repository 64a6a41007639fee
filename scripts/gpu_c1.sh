for v in brick generic; do HJ_STAGE_KERNEL=$v timeout 300 python scripts/c1_probe.py >> gpurun_out/c1_probe.log 2>&1; done
echo done
