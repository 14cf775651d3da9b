cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/umma_probe2 umma_probe2.cu && timeout 60 /tmp/umma_probe2
