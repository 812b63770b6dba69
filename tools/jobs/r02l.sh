set -u
O=gpurun_out; R=r02l
export AQR_CHUNK_COLS=16
N="python tools/cfg5_pipe_narrow.py 64 mgs-hp-row"
timeout 300 $N > $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"catchup_kernel" -s 1 -c 1 -o $O/${R}_catchup $N > $O/${R}_ncu.log 2>&1
echo "rc=$?" >> $O/${R}_narrow.log
N2="python tools/cfg5_narrow.py 64 mgs-hp-row 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trailing_w" -s 33 -c 1 -o $O/${R}_trail $N2 > $O/${R}_ncu2.log 2>&1
echo "rc=$?" >> $O/${R}_narrow.log
