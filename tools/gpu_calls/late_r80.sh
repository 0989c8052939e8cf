mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/late80_torchrun1.log 2>&1; echo "rc=$?" >> gpurun_out/late80_torchrun1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/late80_torchrun1_ref.log 2>&1; echo "rc=$?" >> gpurun_out/late80_torchrun1_ref.log
