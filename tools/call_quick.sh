# quick GPU check: selected tests + attention timing
set -u
O=gpurun_out/${1:-quick}; shift || true
mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 900 python -m pytest ${TESTS:-tests -m gpu} ${KEXPR:+-k "$KEXPR"} -x -q > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
timeout 300 python tools/timeall.py deep32k agentic8k wide > $O/timeall.txt 2>&1
echo done
