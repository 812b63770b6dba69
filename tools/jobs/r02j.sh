set -u
O=gpurun_out; R=${1:-r02j}
mkdir -p $O
export AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so
: > $O/${R}_ab.jsonl
for kv in "4 0" "2 0" "1 0" "2 1" "2 2" "2 3"; do
  set -- $kv
  AQR_XC_ROWS=$1 AQR_SPMM_VARIANT=$2 timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
