# steady-state per-tile cost + L2/DRAM throughput of the fwd and dK/dV kernels (C2)
mkdir -p gpurun_out
for L in 8192 1024; do L=$L B=$((32768/L)) timeout 120 python scripts/steady.py; done
M=gpu__time_duration.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__instruction_throughput.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:hstu --launch-skip 3 -c 3 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/probe_ncu.csv 2>gpurun_out/probe_ncu.err; echo ncu=$?
