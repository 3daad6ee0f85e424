TT_DEBUG_FWD=8 timeout 100 python tools/fwdcount.py 2>&1 | tail -1
sed 's/os.environ\["TT_DEBUG_FWD"\] = "8"/os.environ["TT_DEBUG_FWD"] = "24"/' tools/fwdcount.py > /tmp/fc24.py
timeout 100 python /tmp/fc24.py 2>&1 | tail -1
