timeout 150 python tools/bwdtest.py 2>&1 | tail -4
for d in 0 7; do echo "dbg=$d"; TT_DEBUG_BWD=$d timeout 120 python tools/timeall.py agentic8k deep32k 2>&1 | grep -o "bwd [0-9.]* ms ([0-9]* TF/s)" ; done
