nvidia-smi --query-gpu=serial --format=csv,noheader
for i in 1 2 3 4 5 6; do for c in none 0; do
 if [ $c = none ]; then unset CURAST_CARVEOUT; else export CURAST_CARVEOUT=$c; fi
 python bench.py --steps 200 --warmup 10 --profile 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$c', round(d['ms_per_step'],4), round(d['config']['stage_ms']['stage1'],4), d['clocks'])"
done; done
