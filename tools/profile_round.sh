#!/bin/bash
# Round evidence on one B200 (run under gpurun): the default bench line, the
# steady-state launch list and one `ncu --set full` capture of the top kernels.
# Outputs land in gpurun_out/ (scratch); summaries are copied into profiles/ by
# tools/summarise_round.py <tag>.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1
echo "bench=$?"
C="python bench.py --no-cpu --no-e2e --no-extra --steps 2 --warmup 6"
$C > gpurun_out/plain_l.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 420 -c 140 --csv \
      --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_l.log 2>&1
echo "launches=$?"
C2="python bench.py --no-cpu --no-e2e --no-extra --steps 1 --warmup 6"
$C2 > gpurun_out/plain_f.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"k_ytail|k_vhead_otf|k_uside_tc|k_uside_scatter|k_sel_hist|k_polish" -s 30 -c 10 \
      -o gpurun_out/prof_full $C2 > gpurun_out/ncu_f.log 2>&1
echo "full=$?"
