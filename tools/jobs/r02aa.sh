set -u
O=gpurun_out; R=r02aa
timeout 900 python tools/e2e_repeat.py mgs-hp-row 4 > $O/${R}_e2e.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/${R}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${R}_gpu_tests.log
timeout 1200 python bench.py --no-cpu-baseline > $O/${R}_bench.json 2> $O/${R}_bench.err
