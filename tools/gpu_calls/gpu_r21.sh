mkdir -p gpurun_out
rm -f gpurun_out/r21_ab.jsonl
python tools/s1_ab.py B default:CURAST_CHUNK_MAX=1024:CURAST_CHUNK_MAX=512:CURAST_CHUNK_MAX=256 20 2 >> gpurun_out/r21_ab.jsonl 2>&1
for c in 2048 512; do
CURAST_CHUNK_MAX=$c timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_s1_v2" -s 1 -c 1 --csv python tools/frame_once.py B 1 > gpurun_out/r21_ncu_$c.csv 2>&1
done
