# The N>1 bench path on one GPU (2 ranks sharing it, gloo for the record
# exchange): the JSON line and the shard kernels are what is checked; the
# timing of ranks sharing one GPU means nothing.
mkdir -p gpurun_out
BSSMPPI_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/dist2.log 2>&1
echo "rc=$?" >> gpurun_out/dist2.log
grep -E '^\{|rc=' gpurun_out/dist2.log | cut -c1-400
