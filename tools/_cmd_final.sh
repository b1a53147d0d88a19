set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f_gpu.txt
python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; tail -2 gpurun_out/f_tests.log
timeout 900 python tools/validate_full.py > gpurun_out/f_validate.json 2> gpurun_out/f_validate.err
for c in c1 c2 c3 c4 e1; do timeout 900 python bench.py --config $c > gpurun_out/f_bench_$c.json 2> gpurun_out/f_bench_$c.err; done
for c in c1 c2 c3 c4 e1; do timeout 900 python bench.py --impl reference --config $c --steps 5 --warmup 1 > gpurun_out/f_ref_$c.json 2> gpurun_out/f_ref_$c.err; done
timeout 600 python bench.py --scaling strong --no-cpu-baseline > gpurun_out/f_bench_c1_strong.json 2>/dev/null
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:resample_align -c 1 -o gpurun_out/f_c1 $B --config c1 > /dev/null 2>&1
timeout 900 $N -k regex:srv_align -c 1 -o gpurun_out/f_c4 $B --config c4 > /dev/null 2>&1
timeout 900 $N -k regex:"allpairs_kernel|spectra_kernel" -c 2 -o gpurun_out/f_c2 $B --config c2 > /dev/null 2>&1
timeout 900 $N -k regex:"f1_kernel|fp_kernel|p2_kernel|pick_kernel|stats_partial|aligned_kernel" -c 6 -o gpurun_out/f_c3 $B --config c3 > /dev/null 2>&1
for c in c1 c2 c3 c4 e1; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_${c}_launches.csv $B --config $c > /dev/null 2>&1; done
ls -la gpurun_out/ | tail -40
