export FMM_GEN=device
python tests/sweep_variants.py --config 5 --variants=-1 --iters 2 > gpurun_out/r2b_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fmm_rows -s 2 -c 1 -o gpurun_out/r2b_config5_rows python tests/sweep_variants.py --config 5 --variants=-1 --iters 2 > gpurun_out/r2b_ncu_c5.log 2>&1
echo done
