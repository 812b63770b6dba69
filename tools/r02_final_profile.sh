# Round-2 profile set (run under gpurun): bench line, its ncu launch list,
# full captures of the config-5 kernels on the narrow run and of the DMMA
# block apply.  Every ncu command runs right after the same command exited 0.
set -u
R=${1:-r02i}
O=gpurun_out
mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > $O/${R}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches.csv $CMD > $O/${R}_ncu1.log 2>&1
echo "launch list rc=$?" >> $O/${R}_plain.log
N="python tools/cfg5_narrow.py 64 mgs-hp-row 1"
timeout 300 $N > $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"x_catchup|band_spmm|csr_spmm2" -c 2 -o $O/${R}_c5_x $N > $O/${R}_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trailing_w|col_lazy" -s 40 -c 4 -o $O/${R}_c5_t $N > $O/${R}_ncu3.log 2>&1
echo "captures rc=$?" >> $O/${R}_narrow.log
# the fused HA step on the banded view (config 5's operator, n' = 16, step 4)
NA="python tools/cfg5_narrow.py 16 mgs-ha-row 1"
timeout 300 $NA >> $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_step -s 4 -c 1 -o $O/${R}_c5_s $NA > $O/${R}_ncu5.log 2>&1
echo "ha step rc=$?" >> $O/${R}_narrow.log
timeout 300 python tools/dgemm_bench.py > $O/${R}_dgemm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_dmma -c 1 -o $O/${R}_dmma python tools/dgemm_bench.py > $O/${R}_ncu4.log 2>&1
echo "dmma rc=$?" >> $O/${R}_dgemm.log
