set -u
O=gpurun_out; R=r02x
N="python tools/cfg5_narrow.py 64 mgs-hp-row 1"
timeout 300 $N > $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:x_catchup_stream -c 1 -o $O/${R}_xs $N > $O/${R}_ncu.log 2>&1
echo "rc=$?" >> $O/${R}_narrow.log
N2="python tools/cfg5_narrow.py 64 mgs-ha-row 1"
timeout 300 $N2 >> $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_step_kernel -s 20 -c 1 -o $O/${R}_spmv27 $N2 > $O/${R}_ncu2.log 2>&1
echo "rc=$?" >> $O/${R}_narrow.log
