set -u
O=gpurun_out; R=r02n
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_distributed.py -x -q > $O/${R}_mr.log 2>&1; echo "rc=$?" >> $O/${R}_mr.log
export AQR_CHUNK_COLS=16
N="python tools/cfg5_pipe_narrow.py 64 mgs-hp-row"
timeout 300 $N > $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^catchup_kernel -s 1 -c 1 -o $O/${R}_catchup $N > $O/${R}_ncu.log 2>&1
echo "rc=$?" >> $O/${R}_narrow.log
unset AQR_CHUNK_COLS
timeout 2400 python -m pytest tests -m gpu -x -q > $O/${R}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_gpu_tests.log
