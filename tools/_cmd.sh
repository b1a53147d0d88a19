set -x
python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
for c in c2 c3 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_r2_$c.json 2>&1; done
python bench.py --impl reference > gpurun_out/bench_r2_ref.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resample_align -s 1 -c 1 -o gpurun_out/prof_r2b -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r2b.log 2>&1
cp paper_2501_17779_b200/libcurvalign_cuda.so gpurun_out/prof_r2b.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches_r2_c1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r2.log 2>&1
tail -2 gpurun_out/*.json
