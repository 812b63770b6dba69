set -x
for meth in mgs-ha-row mgs-hp-row; do
AQR_LDG_REVERSE=0 python tools/kernel_ab.py $meth
python tools/kernel_ab.py $meth
for K in 4 8 12 16; do AQR_DEBUG_TIMING= AQR_L2_TAIL=$K python tools/kernel_ab.py $meth; done
AQR_LDG_REVERSE=0 AQR_L2_TAIL=8 python tools/kernel_ab.py $meth
done
AQR_DEBUG_TIMING=1 AQR_L2_TAIL=8 python tools/kernel_ab.py 2>&1 | grep "l2 window"
