set -u
O=gpurun_out; R=r02p
timeout 2000 python tools/e2e_cfg5.py mgs-hp-row 16 -16 32 -32 24 > $O/${R}_e2e.json 2> $O/${R}_e2e.err
