# out-of-core (3 slots, duplex, paired-step order) parity + benches; full GPU suite when FULL=1
if [ "$FULL" = 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_ooc.log 2>&1; echo rc=$? >> gpurun_out/pytest_ooc.log
else
  timeout 1200 python -m pytest tests -m gpu -q -k "out_of_core or host_part or disjoint_rows" > gpurun_out/pytest_ooc.log 2>&1; echo rc=$? >> gpurun_out/pytest_ooc.log
fi
for n in 4 8; do
python bench.py --host-partitions $n --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ooc$n.json 2> gpurun_out/bench_ooc$n.err
done
