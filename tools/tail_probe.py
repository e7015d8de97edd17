import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1711_04556_b200 import SearchParams, synth, decide_static, extract_features
from paper_1711_04556_b200.device import BatchSolver, SolveConfig, WK_FIELDS
NI = int(sys.argv[1]) if len(sys.argv) > 1 else 600
insts = synth.benchmark_batch("j120", NI)
modes = [1] * NI
p = SearchParams.defaults_for(122, total_iters=1000, workers=2, seed=0)
cfg = SolveConfig(total_iters=1000, workers=2, pool_size=16, tabu_size=p.tabu_size, delta=60, phi_steps=20, phi_max=3, seed=0)
s = BatchSolver(insts, modes, cfg)
for rep in range(2):
    s.reset() if rep else None
    r = s.run()
ws = s.w_stats.cpu().numpy()
t0 = ws[:, :, WK_FIELDS['t0']].astype(np.float64); t1 = ws[:, :, WK_FIELDS['t1']].astype(np.float64)
base = t0.min()
ends = (t1 - base) * 1e-6
starts = (t0 - base) * 1e-6
print('device ms', r.device_ms, 'search ms', r.search_ms)
print('worker start ms: max', starts.max())
print('worker end ms: min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f' % tuple(np.percentile(ends, [0, 10, 50, 90, 100])))
print("SM-slot busy fraction (sum of worker spans / (296 slots * makespan))", ((t1 - t0).sum() * 1e-6) / (296 * ends.max()))
