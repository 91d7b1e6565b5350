O=gpurun_out/splitri; mkdir -p $O
for w in 12 s16; do
  VFN_WARPS=$w python tools/chunk_cost_probe.py --fractions 0.03,0.06,0.1,0.13,0.16,0.19,0.22,0.25,0.28,0.32 --reps 2 > $O/cc_late_$w.json 2> $O/cc_late_$w.err
  python - <<PY
import json
d=json.load(open("$O/cc_late_$w.json"))
print("warps $w", [(r["f"], round(r["gather_ms"],1)) for r in d["chunks"] if r["box"]==2])
PY
done
for w in 12 s16; do VFN_WARPS=$w python bench.py --workload c2 --steps 10 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 $w', d['ms_per_step'], d['roofline']['gather_ms'], d['roofline']['frac'])"; done
