for i in $(seq 1 30); do timeout -s KILL 20 python tools/dbg_sssp.py er10d16 16 > /dev/null 2>&1 || { echo "FAIL at $i rc=$?"; exit 1; }; done; echo "30 runs ok"
