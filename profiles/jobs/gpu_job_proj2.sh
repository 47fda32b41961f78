set -u
timeout 300 python profiles/microbench/proj_speed.py 16384 > gpurun_out/proj_speed.txt 2>&1
CTS_PROJ_DBG_TILE_A=1 timeout 300 python profiles/microbench/proj_speed.py 16384 > gpurun_out/proj_speed_tileA.txt 2>&1
