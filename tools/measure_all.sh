# One GPU call: the driver's bench line, the reference arm, and the launch list of the bench
# command (ncu, cold serialised launches: shares only).  Outputs under gpurun_out/.
set -u
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
