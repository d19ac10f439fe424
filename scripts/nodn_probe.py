import os, sys
ROOT="/root/repo"; sys.path[:0]=[ROOT, ROOT+"/tests"]
os.environ["SSB_TIMELINE"]="/tmp/tl_nodn.txt"
import specs, collections
from paper_1412_0595_b200 import synscale as S
spec, mode = specs.config_spec(3, (4+16+1)*256*0.1)
if sys.argv[1] == "nodn":
    spec.populations = [p for p in spec.populations if p.name != "dn"]
    spec.synapses = [g for g in spec.synapses if g.name != "kc_dn"]
sim = S.Simulation(spec, mode, S.EngineOptions(window=256))
sim.step(256*4); sim.sync(); open("/tmp/tl_nodn.txt","w").close()
sim.step(256*16); sim.sync(); sim.kernel_stats()
rows=[l.split() for l in open("/tmp/tl_nodn.txt")]
agg=collections.defaultdict(list)
t0=min(float(r[1]) for r in rows); t1=max(float(r[2]) for r in rows)
for n,a,b in rows: agg[n].append(float(b)-float(a))
print(sys.argv[1], f"{(t1-t0)/16:.1f} us/window", {n: round(sum(v)/len(v),1) for n,v in agg.items()})
