set -x
mkdir -p gpurun_out/r02
for w in c1 c2 c3 c4 tube; do python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02/bench_$w.json 2> gpurun_out/r02/bench_$w.err; done
python bench.py --steps 5 --warmup 3 > gpurun_out/r02/bench_c5.json 2> gpurun_out/r02/bench_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|cub|fft|Radix|Scan" -c 45 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02/launches_c5.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather_tc -c 1 -o gpurun_out/r02/gather_tc_c5 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02/ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather_tc -c 1 -o gpurun_out/r02/gather_tc_c2 python bench.py --workload c2 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02/ncu_c2.log 2>&1
