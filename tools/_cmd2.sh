timeout 900 ncu --set full --clock-control none -k regex:f1_kernel -s 2 -c 1 -o gpurun_out/prof_f1 -f python bench.py --config c3 --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:fp_kernel -s 2 -c 1 -o gpurun_out/prof_fp -f python bench.py --config c3 --steps 1 --warmup 1 > /dev/null 2>&1
