# same-box A/B of release builds: round-2 start (ab_old = c93e53d), first persistent bwd (ab_ce9e0f0), current
set -u
O=gpurun_out/${1:-r2p}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
for d in ab_old ab_ce9e0f0; do (cd $d && python -m paper_2511_00413_b200.build --force > ../$O/build_$d.log 2>&1); done
for r in 1 2; do
  for d in /root/repo /root/repo/ab_old /root/repo/ab_ce9e0f0; do
    TT_ROOT=$d timeout 300 python tools/timeab.py batch64k deep32k:1 agentic8k >> $O/time.txt 2>&1
  done
done
echo done >> $O/time.txt
