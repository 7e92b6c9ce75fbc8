import os, sys
sys.path.insert(0, '/root/repo')
os.environ['TNQVM_TRACE'] = '1'
from paper_2104_10523_b200 import tnqvm as T
from synth import circuits as C
ctx = T.Context(0)
ops, terms = C.qaoa40(0)
circ = T.Circuit.from_oplist(ops)
tot, per = ctx.expectation(circ, terms[:6], per_term=True, dtype=T.C64, restarts=16)
print(tot)
