# cp.async-staged k = 1 step for long banded rows (intermediate build: measured, not kept) vs the gather step.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > $O/band5_tests.log 2>&1
echo "rc=$?" >> $O/band5_tests.log
tail -n 3 $O/band5_tests.log
timeout 1500 python -m pytest tests/test_gpu_variants.py -x -q -k "BAND" > $O/band5_variants.log 2>&1
echo "rc=$?" >> $O/band5_variants.log
tail -n 3 $O/band5_variants.log
E=paper_1703_10440_b200/libaqr_b200_exp.so
for meth in mgs-ha-row mgs-naive-row; do
  for rep in 1 2; do
    for st in 1 2; do
      AQR_LIB_PATH=$E AQR_BAND_STAGE=$st timeout 900 python tools/kernel_ab.py $meth 5 1 2>> $O/band5.err | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('stage=$st', '$meth', 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','spmv_step','col_update') if k in d))" | tee -a $O/band5_ab.txt
    done
  done
done
N="python tools/cfg5_narrow.py 16 mgs-ha-row 1"
timeout 300 $N > $O/band5_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_step -s 4 -c 1 -o $O/r02o_band_step $N > $O/band5_ncu1.log 2>&1
echo "ncu rc=$?" >> $O/band5_narrow.log
