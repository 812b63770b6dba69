# Banded view, second pass: interior fast path of the gather step, cp.async-staged SpMM tiles.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > $O/band4_tests.log 2>&1
echo "rc=$?" >> $O/band4_tests.log
tail -n 3 $O/band4_tests.log
ab() {  # ab METHOD CFG REPS lib...
  meth=$1; cfg=$2; reps=$3; shift 3
  for rep in 1 2; do
    for lib in "$@"; do
      AQR_LIB_PATH=build_ab/libaqr_$lib.so timeout 900 python tools/kernel_ab.py $meth $cfg $reps 2>> $O/band4.err | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', '$meth', $cfg, 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','spmv_step','col_update','block_apply') if k in d))"
    done
  done
}
ab mgs-hp-row 5 1 base new kc16 kc32 rpt2 minb3 | tee -a $O/band4_ab.txt
ab mgs-ha-row 5 1 base new db5 db14 | tee -a $O/band4_ab.txt
ab mgs-ha-row 2 5 base new | tee -a $O/band4_ab.txt
ab mgs-ha-row 3 3 base new | tee -a $O/band4_ab.txt
N="python tools/cfg5_narrow.py 16 mgs-hp-row 1"
timeout 300 $N > $O/band4_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_spmm -c 1 -o $O/r02m_band_spmm $N > $O/band4_ncu2.log 2>&1
N="python tools/cfg5_narrow.py 16 mgs-ha-row 1"
timeout 300 $N >> $O/band4_narrow.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_step -s 4 -c 1 -o $O/r02m_band_step $N > $O/band4_ncu1.log 2>&1
echo "ncu rc=$?" >> $O/band4_narrow.log
