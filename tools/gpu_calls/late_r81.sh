mkdir -p gpurun_out
timeout 1500 python bench.py --mode E --steps 5 --warmup 3 --profile > gpurun_out/late81_E.log 2>&1; echo "rc=$?" >> gpurun_out/late81_E.log
timeout 1500 python bench.py --mode E --e-compressed --steps 5 --warmup 3 --profile > gpurun_out/late81_Eq.log 2>&1; echo "rc=$?" >> gpurun_out/late81_Eq.log
