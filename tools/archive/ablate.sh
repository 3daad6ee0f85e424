for d in 0 1 4 5; do echo "dbg=$d"; TT_DEBUG_BWD=$d timeout 120 python tools/timeall.py deep32k 2>&1 | grep -o "bwd [0-9.]* ms ([0-9]* TF/s)" ; done
