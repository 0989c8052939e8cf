# A/B of CURAST_S1 variants on config B: bash tools/exp_ab.sh ROUNDS VAR1 VAR2 ...
nvidia-smi --query-gpu=serial --format=csv,noheader
R=$1; shift
for i in $(seq $R); do for m in "$@"; do
 CURAST_S1=$m python bench.py --steps 100 --warmup 10 --profile 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); c=d['clocks']; print('$m', round(d['ms_per_step'],4), round(d['config']['stage_ms']['stage1'],4), c['sm_mhz'], {k:v for k,v in c.items() if 'temp' in k})"
done; done
