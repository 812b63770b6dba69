# Short stencils: prefetch of the next owned rows' operands (L1 / L2) in the banded step kernel.
set -u
O=gpurun_out
mkdir -p $O
ab() {  # ab METHOD CFG REPS lib...
  meth=$1; cfg=$2; reps=$3; shift 3
  for rep in 1 2; do
    for lib in "$@"; do
      AQR_LIB_PATH=build_ab/libaqr_$lib.so timeout 900 python tools/kernel_ab.py $meth $cfg $reps 2>> $O/band6.err | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', '$meth', $cfg, 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','spmv_step','col_update','block_apply') if k in d))"
    done
  done
}
ab mgs-ha-row 2 5 base pf1 pf2 | tee -a $O/band6_ab.txt
ab mgs-ha-row 3 3 base pf1 pf2 | tee -a $O/band6_ab.txt
ab mgs-naive-row 3 3 base pf1 pf2 | tee -a $O/band6_ab.txt
