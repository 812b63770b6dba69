# Reduction-tile rows per thread (AQR_BIG_RPT = 8 / 7 / 6: 2048 / 1792 / 1536-row tiles): wave quantization of
# the trailing pass on configs 2 and 3 (512 / 1024 tiles over 296 resident CTAs = 1.73 / 3.46 waves).
set -u
O=gpurun_out
mkdir -p $O
ab() {
  meth=$1; cfg=$2; reps=$3; shift 3
  for rep in 1 2; do
    for lib in "$@"; do
      AQR_LIB_PATH=build_ab/libaqr_$lib.so timeout 900 python tools/kernel_ab.py $meth $cfg $reps 2>> $O/rpt.err | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', '$meth', $cfg, 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','spmv_step','col_update','x_catchup','block_apply') if k in d))"
    done
  done
}
ab mgs-ha-row 2 5 base rpt7 rpt6 | tee -a $O/rpt_ab.txt
ab mgs-ha-row 3 3 base rpt7 rpt6 | tee -a $O/rpt_ab.txt
ab mgs-hp-row 2 5 base rpt7 | tee -a $O/rpt_ab.txt
ab mgs-hp-row 5 1 base rpt7 | tee -a $O/rpt_ab.txt
