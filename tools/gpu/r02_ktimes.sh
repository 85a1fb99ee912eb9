python - <<'PY'
import sys, time
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
t = time.time(); acts = kernel_table(ex, reps=3); print('kernel_table s', time.time() - t)
ks = [k for a in acts for k in a['kernels']]
print('kernels', len(ks), 'sum us', sum(k['us'] for k in ks), 'tensor us', sum(k['us'] for k in ks if k['flops']))
prof = ex.profile(); print('serial action ms', sum(p[0] for p in prof))
for k in sorted(ks, key=lambda k: -k['us'])[:6]: print(round(k['us'],1), k['name'][:90])
PY
