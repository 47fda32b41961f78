set -u
O=gpurun_out/s2t
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt; tail -2 $O/pytest.txt
timeout 300 python bench.py --no-cpu-baseline > $O/bench_decode.json 2>> $O/bench.err
python -c "import json; d=json.loads(open('$O/bench_decode.json').read().strip().splitlines()[-1]); print(round(d['value']), d['roofline']['frac'])"
