# Windowed trailing passes: parity tests, then A/B of the write-back period
# (AQR_TRAIL_WIN, experiments build) and the X catch-up period on configs 5 and 2.
set -u
O=gpurun_out; R=${1:-r02d}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_accuracy.py -x -q > $O/${R}_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_tests.log
EXP=paper_1703_10440_b200/libaqr_b200_exp.so
for W in 1 4 6 8; do
  AQR_LIB_PATH=$EXP AQR_TRAIL_WIN=$W timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/${R}_c5_w$W.json 2>&1
done
AQR_LIB_PATH=$EXP AQR_X_WIN=16 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/${R}_c5_x16.json 2>&1
AQR_LIB_PATH=$EXP AQR_X_WIN=4 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/${R}_c5_x4.json 2>&1
for W in 1 4 6 8; do
  AQR_LIB_PATH=$EXP AQR_TRAIL_WIN=$W timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${R}_c2_w$W.json 2>&1
  AQR_LIB_PATH=$EXP AQR_TRAIL_WIN=$W timeout 600 python bench.py --config 2 --method mgs-hp-row --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${R}_c2hp_w$W.json 2>&1
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/${R}_c5_e2e.json 2>&1
