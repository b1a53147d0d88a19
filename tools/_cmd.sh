python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
for c in c2 c3 c4 e1; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_r2c_$c.json 2>&1; done
python bench.py --impl reference > gpurun_out/bench_r2c_ref.json 2>&1
python bench.py --impl reference --config e1 --steps 5 --warmup 1 > gpurun_out/bench_r2c_ref_e1.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resample_align -s 1 -c 1 -o gpurun_out/prof_r2f -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r2f.log 2>&1
cp paper_2501_17779_b200/libcurvalign_cuda.so gpurun_out/prof_r2f.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_r2f_c1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:elastic_kernel -s 1 -c 1 -o gpurun_out/prof_r2f_e1 -f python bench.py --config e1 --steps 1 --warmup 1 > gpurun_out/ncu_r2f_e1.log 2>&1
for f in gpurun_out/bench_r2c*.json; do echo $f; head -c 300 $f; echo; done
