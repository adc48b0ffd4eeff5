import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W
from paper_2405_18093_b200 import Model, Pipette
w = W.WORKLOADS["C1"]
B, prof = W.workload_inputs(w)
m = w.model
pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
res = pip.search(Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab), w.bs_global, 3, 100, w.seed)
print("ok", res["plan"].latency_s)
