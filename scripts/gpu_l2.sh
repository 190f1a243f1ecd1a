# L2 traffic breakdown per attention kernel (C2)
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --metrics $M --clock-control none -k regex:hstu --launch-skip 3 -c 3 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/l2_ncu.csv 2>gpurun_out/l2_ncu.err; echo ncu=$?
python3 - <<'PY'
import csv
lines=open('gpurun_out/l2_ncu.csv').read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
for d in csv.DictReader(lines[i:]): print(d['Kernel Name'][:22], d['Metric Name'], d['Metric Value'])
PY
