# local-t v2 (deal off the critical path), JD kernels v2, JD-built bench bank + parity spot-check
set -u
O=gpurun_out/s2j
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "jd or layer_grouped or decode or diag or two_streams or mistral" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -3 $O/pytest.txt
timeout 300 python profiles/microbench/jd_speed.py > $O/jd_speed.txt 2>&1; cat $O/jd_speed.txt | tail -2
timeout 600 python bench.py --config decode > $O/bench_decode.json 2>> $O/bench.err
timeout 300 python bench.py --config multi --no-cpu-baseline > $O/bench_multi.json 2>> $O/bench.err
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
cp paper_2407_00066_b200/libcts.so /tmp/keep.so
$NV -DCTS_LOCAL_T=0 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python bench.py --config decode --no-cpu-baseline > $O/bench_decode_old.json 2>> $O/bench.err
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_fused.py > $O/trace_localt.txt 2>&1
cp /tmp/keep.so paper_2407_00066_b200/libcts.so
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['roofline']['frac'] if 'roofline' in d else '', d.get('clocks',{}).get('sm_mhz'), d.get('parity_check'), d.get('config',{}).get('bank_source'))"; done
tail -3 $O/bench.err
