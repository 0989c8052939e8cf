mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -m gpu -p no:cacheprovider -k "config_e or reference_render_context" > gpurun_out/r17_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r17_tests.log
python bench.py --mode E --e-meshes 400 --e-compressed --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r17_benchEc.log 2>&1
python bench.py --mode E --e-meshes 400 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r17_benchE.log 2>&1
python bench.py --mode strong --steps 20 --warmup 3 --no-cpu-baseline --profile > gpurun_out/r17_benchS.log 2>&1
