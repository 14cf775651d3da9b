cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I../../include -I../../paper_2307_00719_b200/csrc -o /tmp/chain_bench chain_bench.cu && /tmp/chain_bench 100 40 > ../../gpurun_out/probe.log 2>&1
cd ../.. 
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_build_table2|k_absorb4|k_spd_inv" -c 6 -o gpurun_out/prof_chain /tmp/chain_bench 100 40 > gpurun_out/ncu_chain.log 2>&1
