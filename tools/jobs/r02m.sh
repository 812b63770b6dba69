set -u
O=gpurun_out; R=r02m
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_accuracy.py -x -q > $O/${R}_tests.log 2>&1; echo "rc=$?" >> $O/${R}_tests.log
timeout 1500 python tools/e2e_cfg5.py mgs-hp-row 0 32 > $O/${R}_e2e.json 2> $O/${R}_e2e.err
export AQR_CHUNK_COLS=16
N="python tools/cfg5_pipe_narrow.py 64 mgs-hp-row"
timeout 300 $N > $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"catchup_kernel<" -s 1 -c 1 -o $O/${R}_catchup $N > $O/${R}_ncu.log 2>&1
echo "rc=$?" >> $O/${R}_narrow.log
