# misc round-2 checks: every entry point on small inputs, the --strong and --weak bench modes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/sanitize_small.py > gpurun_out/sanitize_small.log 2>&1; echo "sanitize_small rc=$?"
python bench.py --strong --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_strong.json 2> gpurun_out/bench_strong.err; echo "strong rc=$?"
python bench.py --weak --gpus 2 --dist-backend gloo --device 0 --steps 3 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_weak2.json 2> gpurun_out/bench_weak2.err; echo "weak2 rc=$?"
python -c "
import json
for f in ('bench_strong', 'bench_weak2'):
    d = json.loads([l for l in open('gpurun_out/%s.json' % f) if l.startswith('{')][-1])
    print(f, d['n_gpus'], d['scaling'], d['config']['workload'], round(d['ms_per_step'], 4), '%.3e' % d['value'], d['result']['key'], d['timing']['step'])
"
tail -3 gpurun_out/sanitize_small.log
