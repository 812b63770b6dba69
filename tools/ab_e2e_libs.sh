# e2e (host-input pipeline) A/B of alternative builds, alternating: bash tools/ab_e2e_libs.sh METHOD lib...
meth=$1; shift
for rep in 1 2; do for lib in "$@"; do
  printf "%-26s " "$lib"
  AQR_LIB_PATH=$lib python bench.py --config 2 --method $meth --no-cpu-baseline --steps 10 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value %.0f e2e %.0f ms_e2e %.2f' % (d['value'], d['e2e']['value'], 64e3/d['e2e']['value']))"
done; done
