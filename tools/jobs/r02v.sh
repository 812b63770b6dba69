set -u
O=gpurun_out; R=r02v
export AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so
for M in 1 0; do
  echo "merge=$M" >> $O/${R}_e2e.log
  AQR_PIPE_MERGE=$M timeout 900 python tools/e2e_repeat.py mgs-hp-row 5 >> $O/${R}_e2e.log 2>&1
done
export AQR_LIB_PATH=build_ab/libaqr_rpt4.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dgemm.py -x -q > $O/${R}_rpt4_tests.log 2>&1; echo "rc=$?" >> $O/${R}_rpt4_tests.log
: > $O/${R}_ab.jsonl
for W in 4 6 8; do
  AQR_TRAIL_WIN=$W timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
AQR_TRAIL_WIN=8 timeout 600 python tools/kernel_ab.py mgs-ha-row 2 5 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
AQR_TRAIL_WIN=4 timeout 600 python tools/kernel_ab.py mgs-ha-row 2 5 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
