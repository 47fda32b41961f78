set -u
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
