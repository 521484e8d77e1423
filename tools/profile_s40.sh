#!/bin/bash
# Round-2 session-4: ncu --set full of the u32 min range kernels (Hash-Min CSC / CSR passes of
# superstep 1, SSSP's first dense pull) with the request metrics, on the library-relabelled cfg4
# graph.  Each command runs once plainly (must exit 0) before it runs under ncu.
set -x
RA="python tools/run_app.py --config cfg4 --relabel"
$RA --app cc > gpurun_out/p_cc.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_pull_ranges" --launch-count 2 -o gpurun_out/cc_full_s40 $RA --app cc > gpurun_out/ncu_cc.log 2>&1
$RA --app sssp > gpurun_out/p_sssp.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_pull_ranges" --launch-count 1 -o gpurun_out/sssp_full_s40 $RA --app sssp > gpurun_out/ncu_sssp.log 2>&1
ls -la gpurun_out/*s40*
