"""Print a slice of the planner tape for ResNet-50g b256 (debugging fusions): tools/tape_dump.py START END."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_net
import paper_1801_04380_b200 as sn
from paper_1801_04380_b200 import _cabi
net=build_net('resnet50g')
cfg=_cabi.sim_config(24<<30, sn.parse_features('liveness,offload,cache,recompute=cost-aware,convselect'), sn.CostConfig(batch=256))
h=_cabi.PlanHandle(net,cfg)
t=h.tape_as_lists()
names={l.id:l.name for l in net.layers}
a,b=int(sys.argv[1]),int(sys.argv[2])
for i in range(a, min(b,len(t))):
    e=t[i]
    if e[0] in 'AF': nm=names.get(e[2])
    else: nm=names.get(e[1])
    print(i,e,nm)
