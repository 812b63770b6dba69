set -u
O=gpurun_out; R=${1:-r02h}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dgemm.py tests/test_gpu_parity.py -x -q > $O/${R}_tests.log 2>&1; echo "rc=$?" >> $O/${R}_tests.log
export AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so
: > $O/${R}_ab.jsonl
for kv in "1 16" "0 16" "1 24" "1 32"; do
  set -- $kv
  AQR_X_SIDE=$1 AQR_X_WIN=$2 timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
unset AQR_LIB_PATH
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/${R}_c5.json 2> $O/${R}_c5.err
timeout 900 python bench.py --config 4 --method mgs-hp-row --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${R}_c4hp.json 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/${R}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_gpu_tests.log
