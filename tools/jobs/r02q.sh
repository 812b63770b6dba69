set -u
O=gpurun_out; R=r02q
export AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so
: > $O/${R}_ab.jsonl
for X in 1 0; do
  AQR_XC_STREAM=$X timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
AQR_PIPE_MERGE=1 timeout 1500 python tools/e2e_cfg5.py mgs-hp-row 16 8 > $O/${R}_e2e_merge.json 2> $O/${R}_e2e.err
AQR_PIPE_MERGE=0 timeout 1500 python tools/e2e_cfg5.py mgs-hp-row 16 > $O/${R}_e2e_nomerge.json 2>> $O/${R}_e2e.err
unset AQR_LIB_PATH
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > $O/${R}_tests.log 2>&1; echo "rc=$?" >> $O/${R}_tests.log
