#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box; one GPU; never multi-rank)
# usage: bash tools/profile.sh [target:kernel-regex ...]   (default: all)
set -x
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu > /dev/null 2>&1
TARGETS=${@:-cfg1:bm_reduce dot:bm_reduce logistic:gemv_n_vec logistic_fused:bm_lgrad gemm_f32:gemm_3xtf32 gemm_f64:gemm_dmma rdim0:rdim0 rdim1:rdim1}
for t in $TARGETS; do
  w=${t%%:*}; k=${t##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $OUT/prof_$w python tools/profile_targets.py $w > $OUT/ncu_$w.log 2>&1
done
ls -la $OUT
