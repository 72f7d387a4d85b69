# ncu --set full of one ring-kernel launch on C2 with n = 1 and n = 8 (one GPU, m parts per rank): red contention check
for m in 1 8; do
  timeout 900 ncu --set full --clock-control none -k regex:sgd_ring -s 2 -c 1 -o gpurun_out/prof_parts_m$m python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/ncu_parts_m$m.log 2>&1
  ncu -i gpurun_out/prof_parts_m$m.ncu-rep --page raw --csv > gpurun_out/prof_parts_raw_m$m.csv 2>&1
  ncu -i gpurun_out/prof_parts_m$m.ncu-rep --page details --csv > gpurun_out/prof_parts_det_m$m.csv 2>&1
  rm -f gpurun_out/prof_parts_m$m.ncu-rep
done
