# Multi-rank bench flow on ONE GPU (tests only): ranks share the device, the
# packed partials travel over gloo through host memory. Validates partitioned
# setup, exchange sizes, eval_begin / exchange / eval_finish and the
# max-over-ranks timing path; the timings themselves are meaningless.
for n in ${NS:-2 4}; do
  TLFEA_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --config ${CFG:-2} --steps 3 --warmup 3 \
    > gpurun_out/multirank_$n.json 2> gpurun_out/multirank_$n.err
  echo "N=$n rc=$? $(head -c 160 gpurun_out/multirank_$n.json)"
done
