# round 2, GPU pass jj: quality of the vertex-tile order on a C4-sized DC-SBM (7.9 M nodes, 8e7 edge draws), n = 1, 20 pools of 2e8 GPU-augmented samples, b = 0 / 14 / 12
set -x
timeout 2400 python tools/quality_vtile.py 7944949 80000000 20 200000000 0,14,12 > gpurun_out/r2jj_quality_c4size.json 2> gpurun_out/r2jj_quality_c4size.err; echo q=$?
tail -4 gpurun_out/r2jj_quality_c4size.err
