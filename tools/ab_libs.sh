# A/B of alternative builds (AQR_LIB_PATH), alternating, step time of config 2
# usage: bash tools/ab_libs.sh METHOD lib1 lib2 ...
meth=$1; shift
for rep in 1 2 3; do
  for lib in "$@"; do
    printf "%-28s " "$lib"
    AQR_LIB_PATH=$lib python tools/kernel_ab.py $meth | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('step %.3f ms  trailing %.3f ms' % (d['step_ms'], d['trailing']['ms_per_fact']))"
  done
done
