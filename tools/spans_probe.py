import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1711_04556_b200 import SearchParams, synth, decide_static, extract_features
from paper_1711_04556_b200.device import BatchSolver, SolveConfig
insts = synth.benchmark_batch('j120', 148)
modes = [int(decide_static(extract_features(x))) for x in insts]
p = SearchParams.defaults_for(122, total_iters=300, workers=2, seed=0)
import os; cfg = SolveConfig(total_iters=300, workers=2, pool_size=16, tabu_size=800, delta=60, phi_steps=20, phi_max=3, seed=0, group=int(os.environ.get("G", "16")), steal=os.environ.get("STEAL", "1") == "1")
s = BatchSolver(insts, modes, cfg)
for rep in range(2):
    s.reset(); r = s.run()
span = r.inst_wall_s
hdr = s.ws_hdr.cpu().numpy(); t0 = hdr[:, 9]; t1 = hdr[:, 10]
print('search_ms', r.search_ms, 'device_ms', r.device_ms)
print('span mean %.3f max %.3f min %.3f' % (span.mean(), span.max(), span.min()))
print('start spread ms', (t0.max() - t0.min()) / 1e6, 'end spread ms', (t1.max() - t1.min()) / 1e6)
ev = r.evaluations - r.pool_evaluations
print('evals per inst mean %.0f max %.0f min %.0f' % (ev.mean(), ev.max(), ev.min()))
print('util (sum span / (n * max))', span.sum() / (len(span) * span.max()))
ws = s.w_stats.cpu().numpy().reshape(-1, 16)
t0w = ws[:, 7]; t1w = ws[:, 8]
tmin = t0w[t0w > 0].min()
ex = (t1w - tmin) / 1e6
print('worker exit ms: min %.0f p10 %.0f median %.0f p90 %.0f max %.0f' % tuple(np.percentile(ex, [0, 10, 50, 90, 100])))
print('exchanges total', int(r.exchanges.sum()), 'mean grant ~', float((r.iterations.sum()) / max(1, r.exchanges.sum())))
