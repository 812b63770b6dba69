# Staged tiles of the banded view: tests, A/B against the gather kernels (experiments build), ncu.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > $O/band3_tests.log 2>&1
echo "rc=$?" >> $O/band3_tests.log
tail -3 $O/band3_tests.log
timeout 1500 python -m pytest tests/test_gpu_variants.py -x -q -k "BAND or SPLIT or knobs0" > $O/band3_variants.log 2>&1
echo "rc=$?" >> $O/band3_variants.log
tail -3 $O/band3_variants.log
E=paper_1703_10440_b200/libaqr_b200_exp.so
for meth in mgs-ha-row mgs-hp-row; do
  for rep in 1 2; do
    for st in 1 0; do
      AQR_LIB_PATH=$E AQR_BAND_STAGE=$st timeout 900 python tools/kernel_ab.py $meth 5 1 2>> $O/band3.err | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('stage=$st', '$meth', 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','spmv_step','col_update','x_catchup','block_apply') if k in d))" | tee -a $O/band3_ab.txt
    done
  done
done
AQR_LIB_PATH=$E AQR_SPLIT_LONG=0 timeout 900 python tools/kernel_ab.py mgs-ha-row 5 1 2>> $O/band3.err | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('stage=1 fused-update', 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','spmv_step','col_update') if k in d))" | tee -a $O/band3_ab.txt
N="python tools/cfg5_narrow.py 16 mgs-ha-row 1"
timeout 300 $N > $O/band3_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_step -s 4 -c 1 -o $O/r02l_band_step $N > $O/band3_ncu1.log 2>&1
N="python tools/cfg5_narrow.py 16 mgs-hp-row 1"
timeout 300 $N >> $O/band3_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_spmm -c 1 -o $O/r02l_band_spmm $N > $O/band3_ncu2.log 2>&1
echo "ncu rc=$?" >> $O/band3_narrow.log
