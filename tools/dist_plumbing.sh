# Plumbing run of bench.py's N>1 path on a one-GPU box: two ranks share the device over gloo
# (host-side collectives only: no kernel waits on another rank).  Not a measurement.
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-suite \
  > gpurun_out/dist2.json 2> gpurun_out/dist2.err; echo dist2=$?
tail -c 1500 gpurun_out/dist2.json; tail -5 gpurun_out/dist2.err
