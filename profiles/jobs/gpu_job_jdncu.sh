set -u
ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:"jd_" -c 14 --csv python profiles/microbench/jd_speed.py 1 > gpurun_out/jd_ncu.csv 2>&1
