# Round-2 bench lines for every workload (profiles/r02/final_*.json)
mkdir -p gpurun_out/r02f
for w in c1 c2 c3 c4 tube; do python bench.py --workload $w --steps 10 --warmup 5 > gpurun_out/r02f/final_$w.json 2> gpurun_out/r02f/final_$w.err; done
python bench.py --steps 10 --warmup 3 > gpurun_out/r02f/final_c5.json 2> gpurun_out/r02f/final_c5.err
for m in 2 3 4 5 7 8; do python bench.py --cutoff $m --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r02f/final_c5_m$m.json 2>&1; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02f/final_reference_c5.json 2>&1
