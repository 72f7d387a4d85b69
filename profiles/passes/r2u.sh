# round 2, GPU pass u: vertex-tile ordering experiment — DRAM bytes of the SGD launches on sorted C5 pools (single-pass ncu metrics), C2 timings
set -x
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sgd_ring -c 6 --csv --log-file gpurun_out/r2u_vtile_c5_dram.csv python tools/exp_vtile.py --shifts none,14,12 --steps 1 > gpurun_out/r2u_vtile_c5_ncu.json 2> gpurun_out/r2u_vtile_c5_ncu.err; echo ncu=$?
timeout 900 python tools/exp_vtile.py --config C2 --shifts none,12,14,16,none > gpurun_out/r2u_vtile_c2.json 2> gpurun_out/r2u_vtile_c2.err; echo c2=$?
