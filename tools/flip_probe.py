import sys, os, json, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2212_14201_b200 import _native as N, qforge as Q
n=28; A=1<<n
sv=Q.StateVector(n); sv.apply_circuit(Q.gen_random_circuit(n,1,7).gates())
L=N.lib(); st=torch.cuda.ExternalStream(L.qs_stream(sv.handle()), device=torch.device('cuda',0))
def t(name, g):
    sv.apply_gate(g); torch.cuda.synchronize(); ts=[]
    for _ in range(5):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(st); sv.apply_gate(g); e1.record(st); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ms=statistics.median(ts); print(name, round(ms,3), round(32*A/(ms/1e3)/1e9/6557,3))
for q in (0, 14, 25, 27):
    t("X q%d"%q, Q.make_gate(Q.GateKind.X,[q]))
    t("H q%d"%q, Q.make_gate(Q.GateKind.H,[q]))
    t("Y q%d"%q, Q.make_gate(Q.GateKind.Y,[q]))
