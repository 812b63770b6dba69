# Banded view: tests, build-variant A/B (step kernel), ncu captures.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > $O/band_tests.log 2>&1
echo "rc=$?" >> $O/band_tests.log
tail -3 $O/band_tests.log
ab() {  # ab METHOD CFG REPS lib...
  meth=$1; cfg=$2; reps=$3; shift 3
  for rep in 1 2; do
    for lib in "$@"; do
      AQR_LIB_PATH=build_ab/libaqr_$lib.so timeout 900 python tools/kernel_ab.py $meth $cfg $reps 2>> $O/band_ab2.err | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', '$meth', $cfg, 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','spmv_step','col_update','block_apply') if k in d))"
    done
  done
}
ab mgs-ha-row 2 5 base u5_3 u5_1 g592 | tee -a $O/band_ab2.txt
ab mgs-ha-row 3 3 base u9_2 g592 | tee -a $O/band_ab2.txt
ab mgs-ha-row 5 1 base db14 db5 g592 | tee -a $O/band_ab2.txt
N="python tools/cfg5_narrow.py 16 mgs-ha-row 1"
timeout 300 $N > $O/band_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_step -s 4 -c 1 -o $O/r02k_band_step $N > $O/band_ncu1.log 2>&1
N="python tools/cfg5_narrow.py 16 mgs-hp-row 1"
timeout 300 $N >> $O/band_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_spmm -c 1 -o $O/r02k_band_spmm $N > $O/band_ncu2.log 2>&1
echo "ncu rc=$?" >> $O/band_narrow.log
