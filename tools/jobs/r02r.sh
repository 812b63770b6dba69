set -u
O=gpurun_out; R=r02r
timeout 1200 python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err
timeout 900 python bench.py --impl reference > $O/${R}_ref.json 2> $O/${R}_ref.err
timeout 2400 python tools/run_configs.py 2 3 4 5 > $O/${R}_configs.jsonl 2> $O/${R}_configs.err
