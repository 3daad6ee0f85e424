for d in 0 32; do echo "dbg=$d"; TT_DEBUG_FWD=$d timeout 100 python tools/timeall.py deep32k agentic8k 2>&1 | grep -o "^[a-z0-9]*: N=[0-9]* fwd [0-9.]* ms ([0-9]* TF/s)"; done
