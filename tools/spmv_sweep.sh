mkdir -p gpurun_out
CMD="python bench.py --steps 10 --warmup 3 --no-suite --no-e2e --no-cpu-baseline"
for W in 64 128 256; do for T in 256 512 1024 2048; do
  echo "W=$W T=$T $(PENCIL_SPMV_WCHUNK=$W PENCIL_SPMV_TILE=$T $CMD | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["value"],1))')" >> gpurun_out/sweep.txt
done; done
echo done
