#!/bin/bash
# Round-2 session-4 profile capture (run under gpurun from the repo root): ncu --set full of the
# flagged PageRank superstep's kernels (superstep 2) on the library-relabelled cfg4 graph, and the
# launch list of bench.py.  Each command runs once plainly (must exit 0) before it runs under ncu.
set -x
RA="python tools/run_app.py --config cfg4 --relabel"
$RA --app pagerank --mode pull --iterations 10 > gpurun_out/p_pr.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_pr_flag|k_flag_fixup|k_pr_finish" --launch-skip 3 --launch-count 3 -o gpurun_out/prf_full_s38 $RA --app pagerank --mode pull --iterations 10 > gpurun_out/ncu_prf.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/b2.json 2> gpurun_out/b2.log && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/bench_launches_s38.csv python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out/*s38*
