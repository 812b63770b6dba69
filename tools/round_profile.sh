# One GPU call: gpu tests, bench lines (HA, HP), the ncu launch list of the
# bench command and full captures of the top kernels (each ncu command runs
# right after the same command exited 0 without ncu).  Outputs in gpurun_out/.
set -u
R=${1:-r01}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${R}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_gpu_tests.log
python bench.py --config 2 > $O/${R}_bench_ha.json 2> $O/${R}_bench_ha.err
python bench.py --config 2 --method mgs-hp-row --no-cpu-baseline > $O/${R}_bench_hp.json 2> $O/${R}_bench_hp.err
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > $O/${R}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches.csv $CMD > $O/${R}_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:trailing_kernel -s 64 -c 3 -o $O/${R}_trailing_early $CMD > $O/${R}_ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:trailing_kernel -s 96 -c 2 -o $O/${R}_trailing_mid $CMD > $O/${R}_ncu3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:csr_step -s 70 -c 2 -o $O/${R}_spmv_full $CMD > $O/${R}_ncu4.log 2>&1
echo "profile rc=$?" >> $O/${R}_plain.log
