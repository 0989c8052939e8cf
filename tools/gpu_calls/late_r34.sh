mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_PROVE=0 20 3 > gpurun_out/late34_ab_B.jsonl 2>&1
python tools/s1_ab.py C default:CURAST_PROVE=0 10 2 > gpurun_out/late34_ab_C.jsonl 2>&1
python tools/s1_ab.py A default:CURAST_PROVE=0 10 2 > gpurun_out/late34_ab_A.jsonl 2>&1
python tools/frame_once.py B 1 > gpurun_out/late34_B_stats.txt 2>&1
