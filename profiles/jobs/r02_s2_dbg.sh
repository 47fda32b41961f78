set -u
O=gpurun_out/s2d
mkdir -p $O
timeout 120 python profiles/microbench/debug_localt.py > $O/debug.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python profiles/microbench/debug_localt.py > $O/memcheck.txt 2>&1
cat $O/debug.txt; grep -m5 -A8 "Invalid\|Error" $O/memcheck.txt | head -60
