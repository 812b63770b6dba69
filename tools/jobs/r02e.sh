# A/B of the write-back period and X catch-up period (experiments build), per-slot times.
set -u
O=gpurun_out; R=${1:-r02e}
mkdir -p $O
export AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so
: > $O/${R}_ab.jsonl
for kv in "4 8" "4 16" "4 24" "4 32" "5 16" "5 24" "6 16" "6 24"; do
  set -- $kv
  AQR_TRAIL_WIN=$1 AQR_X_WIN=$2 timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
for W in 4 5; do
  AQR_TRAIL_WIN=$W timeout 600 python tools/kernel_ab.py mgs-ha-row 2 5 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
  AQR_TRAIL_WIN=$W timeout 600 python tools/kernel_ab.py mgs-ha-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
  for X in 8 16; do
    AQR_TRAIL_WIN=$W AQR_X_WIN=$X timeout 600 python tools/kernel_ab.py mgs-hp-row 2 5 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
  done
done
