# round 2, GPU pass hh: the whole GPU suite on the final source (after the tile-sort slot fix)
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2hh_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/r2hh_gputest.log
