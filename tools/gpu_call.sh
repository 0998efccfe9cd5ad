timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
tail -2 gpurun_out/gputests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['samples_s'], d['check'], d['c4_lsqr']['ms_per_lsqr_iteration'], d['c4_lsqr']['check'], d['c2_dense']['us_per_iteration'])"
