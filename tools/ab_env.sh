# A/B of environment knobs, alternating: bash tools/ab_env.sh METHOD "ENV=a" "ENV=b" ...
export AQR_LIB_PATH=${AQR_LIB_PATH:-paper_1703_10440_b200/libaqr_b200_exp.so}  # knobs: experiments build only
meth=$1; shift
for rep in 1 2 3; do for cfg in "$@"; do
  printf "%-10s %-24s " "$meth" "$cfg"
  env $cfg python tools/kernel_ab.py $meth | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('step %.3f ms  trailing %.3f ms' % (d['step_ms'], d['trailing']['ms_per_fact']))"
done; done
