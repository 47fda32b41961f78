set -u
timeout 900 python -m pytest tests -m gpu -v -x --timeout 120 2>&1 | grep -E "PASS|FAIL|Timeout|Error|error" | tail -20 > gpurun_out/pytest_v.txt
