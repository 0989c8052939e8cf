nvidia-smi --query-gpu=serial --format=csv,noheader
for i in $(seq 1 10); do python tools/kernel_times.py 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print([round(v) for k,v in d['us'].items() if 'lean' in k or 'exact' in k])"; done
