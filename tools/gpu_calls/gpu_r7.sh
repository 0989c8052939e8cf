mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r7_tests.log
for spec in "A superSampling" "C tinyCull" "D instancing" "B base"; do set -- $spec
  if [ "$2" = base ]; then T=""; else T="--toggle $2"; fi
  timeout 900 python -m paper_2604_21749_b200.benchcli $1 $T --frames 60 --output gpurun_out/r7_benchcli_$1_$2.csv > gpurun_out/r7_benchcli_$1_$2.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed
cat > /tmp/res_once.py <<'PY'
import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "tools")
import paper_2604_21749_b200 as cr
from paper_2604_21749_b200.resolve import resolve_frame_device, downsample_device
from frame_once import scene_for
scene, cam = scene_for(sys.argv[1])
dl = cr.build_draw_list(scene, cam)
fb, st = cr.render_draw_list(dl, cam)
for _ in range(3):
    img, rs = resolve_frame_device(fb, dl, cam)
    downsample_device(img, cam.supersampling)
torch.cuda.synchronize()
print(rs)
PY
for c in B A A4; do
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_resolve|k_downsample" -s 2 -c 2 --csv python /tmp/res_once.py $c > gpurun_out/r7_ncu_resolve_$c.csv 2> gpurun_out/r7_ncu_resolve_$c.err
done
