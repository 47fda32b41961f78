set -u
O=gpurun_out/s2k
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "layer_grouped or decode or diag or two_streams or mistral or exclusive" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -2 $O/pytest.txt
for i in 1 2; do
timeout 300 python bench.py --config decode --no-cpu-baseline > $O/bench_decode_$i.json 2>> $O/bench.err
timeout 300 python bench.py --config multi --no-cpu-baseline > $O/bench_multi_$i.json 2>> $O/bench.err
done
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
cp paper_2407_00066_b200/libcts.so /tmp/keep.so
$NV -DCTS_LOCAL_T=0 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
for i in 1 2; do
timeout 300 python bench.py --config decode --no-cpu-baseline > $O/bench_decode_old_$i.json 2>> $O/bench.err
timeout 300 python bench.py --config multi --no-cpu-baseline > $O/bench_multi_old_$i.json 2>> $O/bench.err
done
cp /tmp/keep.so paper_2407_00066_b200/libcts.so
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), d.get('clocks',{}).get('sm_mhz'))"; done
