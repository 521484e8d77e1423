#!/bin/bash
# Round-2 profile capture (run under gpurun from the repo root): ncu --set full of the
# superstep kernels on the library-relabelled cfg4 graph, and the launch list of bench.py.
# Each command runs once plainly (must exit 0) before the same command under ncu.
set -x
RA="python tools/run_app.py --config cfg4 --relabel"
$RA --app pagerank --mode pull --iterations 10 > gpurun_out/p_pr.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_pull_ranges|k_pull_fixup|k_pr_finish" --launch-count 3 -o gpurun_out/pr_full_s33 $RA --app pagerank --mode pull --iterations 10 > gpurun_out/ncu_pr.log 2>&1
$RA --app cc > gpurun_out/p_cc.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_pull_ranges" --launch-count 2 -o gpurun_out/cc_full_s33 $RA --app cc > gpurun_out/ncu_cc.log 2>&1
$RA --app sssp > gpurun_out/p_sssp.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_pull_ranges|k_expand" --launch-skip 1 --launch-count 5 -o gpurun_out/sssp_full_s33 $RA --app sssp > gpurun_out/ncu_sssp.log 2>&1
python bench.py --steps 2 --warmup 3 > gpurun_out/b2.json 2> gpurun_out/b2.log && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/bench_launches_s33.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out/*s33*
