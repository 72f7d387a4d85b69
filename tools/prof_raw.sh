# ncu --set full of the ring kernel (LDGSTS default and TMA variant), raw + SASS source pages as CSV
for v in def tma; do
  if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/prof_raw_$v python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/ncu_raw_$v.log 2>&1
  ncu -i gpurun_out/prof_raw_$v.ncu-rep --page raw --csv > gpurun_out/prof_raw_$v.csv 2>&1
  ncu -i gpurun_out/prof_raw_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_src_$v.csv 2>&1
  ncu -i gpurun_out/prof_raw_$v.ncu-rep --page details --csv > gpurun_out/prof_det_$v.csv 2>&1
  rm -f gpurun_out/prof_raw_$v.ncu-rep
done
