set -u
O=gpurun_out; R=r02o
timeout 2000 python tools/e2e_cfg5.py mgs-hp-row 0 16 -8 -32 > $O/${R}_e2e.json 2> $O/${R}_e2e.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/${R}_c5.json 2> $O/${R}_c5.err
