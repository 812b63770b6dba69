set -u
O=gpurun_out; R=r02b
timeout 1800 python -m pytest tests -m gpu -x -q > $O/${R}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > $O/${R}_bench.json 2> $O/${R}_bench.err
N="python tools/cfg5_narrow.py 32 mgs-hp-row 2"
timeout 300 $N > $O/${R}_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_lazy|trailing" -s 40 -c 4 -o $O/${R}_c5_lazy $N > $O/${R}_ncu2.log 2>&1
echo "captures rc=$?" >> $O/${R}_narrow.log
