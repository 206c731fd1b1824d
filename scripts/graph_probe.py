"""Profiling helper: one density step (SlabRunner, 1 GPU) eager vs replayed from a CUDA graph
(usage: python scripts/graph_probe.py c3).  Prints ms per step of each and whether the outputs
match."""
import sys, time, json
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch, synth
import paper_1804_06231_b200 as pv
from paper_1804_06231_b200 import slabs
pv.load()
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
p = synth.make(cfg)
r = slabs.SlabRunner(slabs.Slab.single(p))
r.upload()
for _ in range(3):
    r.step()
torch.cuda.synchronize()
s = torch.cuda.current_stream()
def t(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
ms_eager = t(r.step)
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(s)
with torch.cuda.stream(cs):
    r.step()
s.wait_stream(cs)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    r.step()
torch.cuda.synchronize()
ref = r.out.rho.clone()
ms_graph = t(g.replay)
g.replay(); torch.cuda.synchronize()
print(json.dumps({"cfg": cfg, "ms_eager": ms_eager, "ms_graph": ms_graph, "same": bool(torch.equal(ref, r.out.rho))}))
