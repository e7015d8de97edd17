#!/usr/bin/env python3
"""Build-container only (needs /root/reference): the reference package itself
(numba backend, all host threads) against the C port the bench uses as its
reference arm, on Gen-P j120 instances.  The port is the faster of the two,
so the bench's GPU/CPU ratios are conservative."""
import sys, time, os
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/reference/pkg/src')
import numpy as np
import oracle
from paper_1711_04556_b200 import synth
import rcpsp_tabu as R
from rcpsp_tabu.cooperation import orchestrate as rorch
from rcpsp_tabu.search import SearchParams as RSP
from rcpsp_tabu.selector import EvalMode as REM
for k in (5, 305, 455):
    inst = synth.benchmark_batch('j120p', 1, first_seed=k)[0]
    rinst = R.make_instance(inst.name, list(map(int, inst.durations)), list(map(int, inst.capacities)),
                            np.asarray(inst.demands).tolist(), [list(s) for s in inst.successors])
    W = os.cpu_count()
    p = RSP.defaults_for(rinst.n_activities, total_iters=300, workers=W, seed=0)
    rorch(rinst, RSP.defaults_for(rinst.n_activities, total_iters=5, workers=1, seed=0), REM.TIME)  # jit warm-up
    t = time.perf_counter(); rs = rorch(rinst, p, REM.TIME); tr = time.perf_counter() - t
    t = time.perf_counter(); os_ = oracle.orchestrate(inst, 300, W, 0, 1); to = time.perf_counter() - t
    print(k, 'numba', round(rs.evaluations / tr / 1e6, 3), 'M/s', 'port', round(os_['evaluations'] / to / 1e6, 3), 'M/s', 'ratio port/numba %.2f' % ((os_['evaluations'] / to) / (rs.evaluations / tr)), 'threads', W)
