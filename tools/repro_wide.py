import sys; sys.path.insert(0, '.')
from paper_1711_04556_b200 import synth
from paper_1711_04556_b200.device import BatchSolver, SolveConfig
mode, cl = int(sys.argv[1]), int(sys.argv[2])
wide = synth.random_instance(50, 6, seed=91, cap_lo=20, cap_hi=60, max_dur=45, demand_density=0.6)
cfg = SolveConfig(total_iters=60, workers=1, pool_size=8, tabu_size=250, delta=60,
                  phi_steps=20, phi_max=3, seed=5, collect_trace=True, cluster=cl)
r = BatchSolver([wide], [mode], cfg).run()
print(mode, cl, r.best_cmax.tolist(), r.evaluations.tolist())
