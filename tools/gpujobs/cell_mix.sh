nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cell_mix tools/micro/cell_mix.cu > /dev/null 2>&1 && /tmp/cell_mix
