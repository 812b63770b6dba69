# Re-entry GPU call: gpu tests, config-5 bench line, launch list of the
# bench command, trailing/lazy captures on the narrow run, and
# compute-sanitizer on the small-shape sweep.  Outputs in gpurun_out/.
set -u
R=${1:-r02c}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current --format=csv > $O/${R}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > $O/${R}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > $O/${R}_bench.json 2> $O/${R}_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > $O/${R}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches.csv $CMD > $O/${R}_ncu1.log 2>&1
echo "launch list rc=$?" >> $O/${R}_plain.log
N="python tools/cfg5_narrow.py 32 mgs-hp-row 2"
timeout 300 $N > $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_lazy|trailing|csr_spmm2|csr_row" -s 40 -c 6 -o $O/${R}_c5 $N > $O/${R}_ncu2.log 2>&1
echo "captures rc=$?" >> $O/${R}_narrow.log
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_small.py > $O/${R}_sanitize_$T.log 2>&1
  echo "rc=$?" >> $O/${R}_sanitize_$T.log
done
