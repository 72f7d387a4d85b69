# round 2, GPU pass ll: the whole GPU suite on the final library (after the GV_VTILE_HINT=2 option)
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2ll_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/r2ll_gputest.log
