mkdir -p gpurun_out
timeout 900 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --import-source on --clock-control none -k regex:dkv --launch-skip 1 -c 1 -o gpurun_out/dkv -f python scripts/trace_c2.py 0 > gpurun_out/ncu_dkv.log 2>&1; echo ncu=$?
tail -5 gpurun_out/ncu_dkv.log
