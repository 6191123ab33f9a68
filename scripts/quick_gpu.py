import sys, time, math, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2010_02857_b200 import ifgf, inputs
name = sys.argv[1]
c = inputs.CONFIGS[name]
pts = c.points(); a = c.densities()
dp = torch.from_numpy(pts).cuda(); da = torch.from_numpy(a).cuda()
t = time.time(); plan = ifgf.Plan(dp, c.k, c.levels, c.Ps, c.Pang); torch.cuda.synchronize(); print(name, 'plan s', time.time()-t, flush=True)
st = plan.stats(); print({k: st[k] for k in ('nseg','near_pairs','s2c_pairs','cousin_evals','upward_evals','plan_device_bytes','plan_ms')}, flush=True)
plan.profile_enable(True)
out = plan.apply(da); torch.cuda.synchronize()
plan.profile_read(reset=True)
ts=[]
for i in range(3):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); out = plan.apply(da); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print('apply ms', ts, 'pts/s', c.n/(min(ts)*1e-3), flush=True)
print(plan.profile_read(), flush=True)
tg = inputs.error_targets(c.n, 1000)
ex = ifgf.direct(dp, c.k, da, torch.from_numpy(tg).cuda()).cpu().numpy()
g = out.cpu().numpy()[tg]
print('rel err vs direct', np.sqrt(np.sum(np.abs(g-ex)**2)/np.sum(np.abs(ex)**2)), flush=True)
print("dfma", ifgf.bench_dfma(20000)); print("dmma", ifgf.bench_dmma(20000))
