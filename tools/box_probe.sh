#!/bin/bash
# Host facts of the GPU box (RAM, cores, MPS, PCIe) for sizing the bench legs.
free -g; nproc; cat /proc/cpuinfo | grep "model name" | head -1
which nvidia-cuda-mps-control nvidia-smi; ls /usr/bin | grep -i nvidia
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv
nvidia-smi -q | grep -i -A3 "compute mode"
