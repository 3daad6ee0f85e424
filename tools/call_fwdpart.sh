set -u
O=gpurun_out/${1:-fwdpart}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
for d in 0 64; do echo "dbg=$d"; TT_DEBUG_FWD=$d timeout 120 python tools/timefwd.py 2>&1; done > $O/ablate.txt
echo done
