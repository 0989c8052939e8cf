# Round-end evidence: GPU tests, smoke, bench line, reference arm, launch list,
# ncu --set full of the stage-1 kernels (traffic), configs table.
# usage: bash tools/gpu_final.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/${T}_clocks.csv &
SMI=$!
python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.log
kill $SMI
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_reference.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1_v2|k_s1_exact" -s 2 -c 2 -o gpurun_out/${T}_stage1_full python tools/frame_once.py B 1 > gpurun_out/${T}_ncu_full.log 2>&1
python tools/configs.py A B C D Bq Dq E200 A4 > gpurun_out/${T}_configs.jsonl 2> gpurun_out/${T}_configs.err
