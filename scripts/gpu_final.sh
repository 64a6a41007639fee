# GPU suite, then the evidence pass without its own suite run (one gpurun call)
TAG=${1:-fin}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_gputests.log
SKIP_TESTS=1 bash scripts/gpu_evidence.sh $TAG
