set -u
O=gpurun_out; R=${1:-r02f}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dgemm.py -x -q > $O/${R}_dgemm_tests.log 2>&1; echo "rc=$?" >> $O/${R}_dgemm_tests.log
timeout 600 python tools/dgemm_bench.py > $O/${R}_dgemm_bench.log 2>&1; echo "rc=$?" >> $O/${R}_dgemm_bench.log
timeout 900 python bench.py --config 4 --method mgs-hp-row --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${R}_c4hp.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_dmma -c 1 -o $O/${R}_dmma python tools/dgemm_bench.py > $O/${R}_ncu_dmma.log 2>&1
N="python tools/cfg5_narrow.py 32 mgs-hp-row 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"csr_spmm2|x_catchup|trailing_w" -c 4 -o $O/${R}_c5 $N > $O/${R}_ncu_c5.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${R}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_gpu_tests.log
