set -u
O=gpurun_out; R=${1:-r02g}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dgemm.py tests/test_gpu_parity.py -x -q > $O/${R}_tests.log 2>&1; echo "rc=$?" >> $O/${R}_tests.log
timeout 600 python tools/dgemm_bench.py > $O/${R}_dgemm_bench.log 2>&1; echo "rc=$?" >> $O/${R}_dgemm_bench.log
export AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so
: > $O/${R}_ab.jsonl
for kv in "4 2 4" "4 2 0" "4 2 2" "4 2 8" "4 4 4" "6 4 4" "8 4 4"; do
  set -- $kv
  AQR_TRAIL_WIN=$1 AQR_TRAIL_CU=$2 AQR_SPMM_SG=$3 timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
for kv in "4 2" "4 4" "6 4" "8 4"; do
  set -- $kv
  AQR_TRAIL_WIN=$1 AQR_TRAIL_CU=$2 timeout 600 python tools/kernel_ab.py mgs-ha-row 2 5 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
unset AQR_LIB_PATH
timeout 1500 python -m pytest tests/test_gpu_variants.py -x -q > $O/${R}_variants.log 2>&1; echo "rc=$?" >> $O/${R}_variants.log
