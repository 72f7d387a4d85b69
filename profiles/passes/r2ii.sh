# round 2, GPU pass ii: the default bench command as the driver runs it (final bench.py: oracle arms with the same vertex tile), and the reference arm
set -x
timeout 1800 python bench.py > gpurun_out/r2ii_bench.json 2> gpurun_out/r2ii_bench.err; echo bench=$?
timeout 1500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2ii_reference.json 2> gpurun_out/r2ii_reference.err; echo reference=$?
