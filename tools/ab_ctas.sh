# trailing-pass column grouping (AQR_TRAIL_CTAS) A/B with per-launch times
export AQR_LIB_PATH=${AQR_LIB_PATH:-paper_1703_10440_b200/libaqr_b200_exp.so}  # knobs: experiments build only
meth=${1:-mgs-ha-row}
for c in 4 2 3 6 8; do
  echo "== AQR_TRAIL_CTAS=$c"
  AQR_TRAIL_CTAS=$c AQR_LIST=1 python tools/kernel_ab.py $meth > /tmp/l.txt 2>&1
  head -1 /tmp/l.txt | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('step %.3f ms  trailing %.3f ms' % (d['step_ms'], d['trailing']['ms_per_fact']))"
  awk '/^launch/ {i=$2+0; us=$4; if (i<16) a+=us; else if (i<48) b+=us; else c+=us} END {printf "launches 0-15 %.0f us, 16-47 %.0f us, 48-63 %.0f us\n", a, b, c}' /tmp/l.txt
done
