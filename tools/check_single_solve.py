import sys; sys.path.insert(0,'.')
import numpy as np, time
from paper_1711_04556_b200 import synth, SearchParams, orchestrate, EvalMode
import oracle
for cfg in ['act300', 'j30']:
    inst = synth.benchmark_batch(cfg, 1, first_seed=2)[0]
    for mode in (EvalMode.TIME, EvalMode.CAPACITY):
        p = SearchParams.defaults_for(inst.n_activities, total_iters=60, workers=1, seed=0, mode=mode, collect_trace=True)
        st = orchestrate(inst, p)
        want = oracle.orchestrate(inst, 60, 1, 0, int(mode), collect_trace=True)
        ok = st.best_cmax == want['best_cmax'] and st.evaluations == want['evaluations'] and [t.tolist() for t in st.traces] == [t.tolist() for t in want['traces']]
        print(cfg, mode.name, st.best_cmax, st.evaluations, 'match' if ok else 'MISMATCH', round(st.wall_time, 3))
