mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2508_04711_b200/csrc scripts/tmem_bw.cu -o /tmp/tmem_bw && timeout 120 /tmp/tmem_bw
bash scripts/gpu_run1.sh
