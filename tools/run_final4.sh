# full GPU suite, default bench (pipeline detail), sampler-thread ablation
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_final4.log 2>&1; echo rc=$? >> gpurun_out/pytest_final4.log
python bench.py > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err
timeout 900 python tools/ablations.py --parts threads --out gpurun_out/next2_threads.json > gpurun_out/next2_threads.log 2>&1
