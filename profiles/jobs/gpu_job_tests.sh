set -u
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -k "bench_configuration or full_size" 2>&1 | tail -15 > gpurun_out/pytest_full.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
