#!/usr/bin/env python3
"""CPU arm variants on the host: instances one after another with all threads
each (the reference's bench, the CPU arm) vs all instances at once with one
thread each.  Build container or GPU box."""
import sys, time, threading, os
sys.path.insert(0,'/root/repo')
import oracle
from paper_1711_04556_b200 import synth
C = os.cpu_count()
insts = [synth.benchmark_batch('j120p',1,first_seed=(k*157)%600)[0] for k in range(C)]
# (a) reference-style: instances one after another, C threads each
t=time.perf_counter(); ev=0
for x in insts[:4]:
    r=oracle.orchestrate(x, 300, C, 0, 1); ev+=r['evaluations']
ta=time.perf_counter()-t; print('sequential instances, %d threads each: %.3f M/s' % (C, ev/ta/1e6))
# (b) instance-parallel: C instances at once, 1 thread each
res=[None]*C
def run(i): res[i]=oracle.orchestrate(insts[i], 300, 1, 0, 1)
t=time.perf_counter(); th=[threading.Thread(target=run,args=(i,)) for i in range(C)]
[x.start() for x in th]; [x.join() for x in th]
tb=time.perf_counter()-t; ev=sum(r['evaluations'] for r in res)
print('instance-parallel, %d instances x 1 thread: %.3f M/s' % (C, ev/tb/1e6))
