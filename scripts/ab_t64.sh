bash scripts/ab_builds.sh abb4 t64
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/abb4_tests.log 2>&1; echo "rc $?" >> gpurun_out/abb4_tests.log
HJ_LIB=check timeout 900 python scripts/bounds_check.py > gpurun_out/abb4_bounds.txt 2>&1; echo "rc $?" >> gpurun_out/abb4_bounds.txt
