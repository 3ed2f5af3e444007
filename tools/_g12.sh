O=gpurun_out/t12; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench=$?" >> $O/status
cat $O/status; tail -3 $O/pytest.log
python3 -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['e2e']['pageable'])
print([r for r in d['records']['rows'] if r[3]=='gpu_sm100' and r[1]==1024])"
