#!/bin/bash
# Reproduce the committed profiles (run on a B200 via gpurun, one GPU):
#   gpurun --timeout 1800 -- 'bash profiles/capture.sh r01'
# Writes gpurun_out/<tag>_*; summaries are extracted with profiles/summarize.py.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu"
export FMM_GEN=device  # R-MAT graphs built on the GPU (same CSR as the host builder)
# 1) plain run of the exact command that ncu will wrap (must exit 0 first)
$BENCH > $OUT/${TAG}_plain.log 2>&1 || { echo "plain bench failed"; exit 1; }
# 2) launch list: every kernel of the bench command with its device time
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_ncu_launches.log 2>&1
# 3) full capture of the top kernel (config 2, the bench workload)
ncu --set full --clock-control none --import-source on -k regex:fmm_rows -s 3 -c 1 \
    -o $OUT/${TAG}_config2_rows $BENCH > $OUT/${TAG}_ncu_c2.log 2>&1
# 4) the other configs' kernels through the sweep tool
for c in 3 4 1 5; do
  python tests/sweep_variants.py --config $c --variants=-1 --iters 3 > $OUT/${TAG}_plain_c$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:fmm_rows -s 3 -c 1 \
      -o $OUT/${TAG}_config${c}_rows python tests/sweep_variants.py --config $c --variants=-1 --iters 3 \
      > $OUT/${TAG}_ncu_c$c.log 2>&1
done
echo capture done
