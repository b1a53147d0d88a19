timeout 900 ncu --set full --clock-control none --import-source on -k regex:srv_align_kernel -s 1 -c 1 -o gpurun_out/prof_c4 -f python bench.py --config c4 --steps 1 --warmup 1 > /dev/null 2>&1
cp paper_2501_17779_b200/libcurvalign_cuda.so gpurun_out/prof_c4.so
