mkdir -p gpurun_out
for sm in 128 64 32 16; do python tools/ktimes_cfg.py C small_max_px=$sm 2>/dev/null | grep "^{" >> gpurun_out/late45_kt.jsonl; done
for sm in 128 16; do python tools/ktimes_cfg.py A small_max_px=$sm 2>/dev/null | grep "^{" >> gpurun_out/late45_kt.jsonl; done
