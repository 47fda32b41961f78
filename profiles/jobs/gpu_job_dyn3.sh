set -u
timeout 600 python -m pytest tests -m gpu -v -x --timeout 60 --timeout-method=thread 2>&1 | grep -E "PASS|FAIL|Timeout|rror" | tail -6 > gpurun_out/pytest_v.txt
for i in 1 2 3 4 5; do
CTS_EXPAND_DYNAMIC=1 timeout 120 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -k "q_proj_r64 or ranks_and_ragged" 2>&1 | tail -1 >> gpurun_out/pytest_loop.txt
done
