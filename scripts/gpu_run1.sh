# GPU iteration: gpu tests, bench, launch list, C2 timeline trace (stops at the first failure)
mkdir -p gpurun_out
rm -f gpurun_out/bench.json gpurun_out/launches.csv gpurun_out/trace_cta0.json
timeout 600 python -u -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest.log 2>&1; rc=$?
tail -15 gpurun_out/pytest.log
[ $rc -eq 0 ] || exit 1
timeout 300 python -u bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?
echo bench=$rc; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
[ $rc -eq 0 ] || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hstu --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-max-len > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 120 python -u scripts/trace_c2.py 0 2>&1 | tail -3
