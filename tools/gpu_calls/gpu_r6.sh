mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r6_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r6_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r6_bench.log
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r6_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r6_ref.log
python bench.py --mode E --e-meshes 200 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6_benchE.log 2>&1; echo "rc=$?" >> gpurun_out/r6_benchE.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r6_launches.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/r6_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1_v2|k_s1_exact" -s 2 -c 2 -o gpurun_out/r6_stage1_full python tools/frame_once.py B 1 > gpurun_out/r6_ncu_full.log 2>&1
