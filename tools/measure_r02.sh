# One GPU call (round 2): smoke(), the GPU suite, the driver's bench line, the reference arm, the
# launch list of the bench command with DRAM bytes per launch (ncu; cold serialised launches:
# shares only) -> profiles/ncu_traffic.json candidates.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
fi
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
if [ "${SKIP_NCU:-0}" != 1 ]; then
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --suite-steps 1 > gpurun_out/bench_small.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --suite-steps 1 > gpurun_out/ncu_bench.log 2>&1
  echo ncu=$?
  python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
  python tools/traffic_capture.py gpurun_out/launches.csv gpurun_out/ncu_traffic.json > /dev/null 2>&1
fi
