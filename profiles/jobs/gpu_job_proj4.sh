set -u
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "projection" 2>&1 | tail -3 > gpurun_out/pytest_proj.txt
CTS_PROJ_A=0 timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "projection" 2>&1 | tail -3 >> gpurun_out/pytest_proj.txt
for a in 1 0; do
CTS_PROJ_A=$a timeout 300 python profiles/microbench/proj_speed.py 16384 > gpurun_out/proj_speed_a$a.txt 2>&1
done
