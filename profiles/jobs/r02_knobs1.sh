# apply_local timing knobs: which part of the decode launch costs what
set -u
mkdir -p gpurun_out
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
run() {  # tag, defines
  $NV $2 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
  timeout 300 python bench.py --config decode --steps 50 --no-cpu-baseline > gpurun_out/knob_$1.json 2>> gpurun_out/knob.err
  python -c "import json; d=json.loads(open('gpurun_out/knob_$1.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['roofline']['avg_launch_us'],1))" >> gpurun_out/knobs.txt
}
run base ""
run noscatter "-DCTS_LOC_NO_SCATTER=1"
run noymath "-DCTS_LOC_NO_YMATH=1"
run noboth "-DCTS_LOC_NO_SCATTER=1 -DCTS_LOC_NO_YMATH=1"
run s70 "-DCTS_LOC_SFRAC=70"
run s25 "-DCTS_LOC_SFRAC=25"
cat gpurun_out/knobs.txt
