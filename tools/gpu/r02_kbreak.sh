# per-kernel replay times of one ResNet-50g b256 iteration, grouped
python - <<'PY' > gpurun_out/kbreak.txt 2>&1
import sys, json, collections
sys.path.insert(0, '.')
import paper_1801_04380_b200 as sn
from paper_1801_04380_b200.training import Executor
from paper_1801_04380_b200.profiling import kernel_table
from bench import build_net, _inputs
net = build_net('resnet50g')
cfg = sn.SimConfig(pool_bytes=24 << 30, features=sn.parse_features('liveness,offload,cache,recompute=cost-aware,convselect'), cost=sn.CostConfig(batch=256))
ex = Executor(net, cfg)
ex.set_inputs(*_inputs(net, 256))
for _ in range(3): ex.step(update=False)
acts = kernel_table(ex, reps=3)
json.dump(acts, open('gpurun_out/kbreak.json', 'w'))
cat = collections.Counter()
rows = []
for a in acts:
    for k in a['kernels']:
        short = k['name'].split('(')[0].replace('(anonymous namespace)::', '').replace('void ', '')[-48:]
        key = (a.get('kind', '-'), a['type'], short)
        cat[key] += k['us']
        rows.append((k['us'], a.get('name', '-'), a['type'], short, a.get('gemm')))
tot = sum(cat.values())
print('total us', round(tot, 1))
for (kind, typ, nm), us in cat.most_common(40):
    print(f'{us:9.1f} {100*us/tot:5.1f}%  {kind:6s} {typ:7s} {nm}')
print()
for r in sorted(rows, key=lambda r: -r[0])[:40]:
    print(f'{r[0]:8.1f}  {r[1]:14s} {r[2]:7s} {r[3]:48s} {r[4]}')
PY
