set -u
timeout 600 python profiles/microbench/jd_speed.py 10 > gpurun_out/jd_speed.txt 2>&1
timeout 600 python profiles/microbench/jd_speed.py 50 >> gpurun_out/jd_speed.txt 2>&1
