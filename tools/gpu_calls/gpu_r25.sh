mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
rm -f gpurun_out/r25_ab.jsonl
for c in D Dq; do python tools/s1_ab.py $c CURAST_LIB=$R/libH.so:CURAST_LIB=$R/libN.so 10 2 >> gpurun_out/r25_ab.jsonl 2>&1; done
