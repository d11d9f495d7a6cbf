# Stroop/DDM-grid/Ext-Stroop launch shape A/B (trial chunks) through the bench extras
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_new.json 2>/dev/null
python -c "
import json
d = json.loads([l for l in open('gpurun_out/ab_new.json') if l.startswith('{')][-1])
a = d['also']
print('stroop_cfg4 ms', a['stroop_cfg4']['ms'], 'ext ms', a['ext_stroop_a']['ms'], 'ddm_grid ms', a['ddm_grid']['ms'])
"
