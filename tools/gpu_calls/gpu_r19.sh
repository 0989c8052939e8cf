mkdir -p gpurun_out
export CURAST_BENCH_SHARED_GPU=1
for m in B strong; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --mode $m --grid-n 3000 > gpurun_out/r19_bench2_$m.log 2>&1; echo "rc=$?" >> gpurun_out/r19_bench2_$m.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --grid-n 2000 > gpurun_out/r19_ref2.log 2>&1; echo "rc=$?" >> gpurun_out/r19_ref2.log
