# A/B: reduction dependents triggered after the streaming phase (default) vs at kernel start
OUT=gpurun_out
: > $OUT/early.txt
for round in 1 2 3; do
for e in 0 1; do
  echo "== early=$e" >> $OUT/early.txt
  BM_EARLY_TRIGGER=$e timeout 300 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $OUT/early.txt 2>&1
done
done
BM_EARLY_TRIGGER=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py -x -q -k "accu or dot or reduce or norm" -p no:cacheprovider >> $OUT/early.txt 2>&1; echo "pytest early rc=$?" >> $OUT/early.txt
