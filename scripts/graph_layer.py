"""Config-2 layer: direct launches vs CUDA-graph replay (same buffers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_19427_b200 import Context

dev = torch.device("cuda:0")
ctx = Context(0)
s = bench.make_workload(torch, dev, 64, 4096)
stream = torch.cuda.Stream()


def layer(i, st):
    k, v = s["kv"][i % bench.N_ROT]
    ctx.mfa_layer(s["w"], s["x"], k, v, s["block_table"], s["seq_lens"], s["h_res"], s["h_norm"], stream=st)


def timed(fn, n=30):
    with torch.cuda.stream(stream):
        for i in range(5):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(n):
            fn(i)
        b.record(stream)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


print("direct us/layer", timed(lambda i: layer(i, stream.cuda_stream)))
graphs = []
for r in range(bench.N_ROT):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        layer(r, stream.cuda_stream)  # warm (workspace, tensor maps)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            layer(r, torch.cuda.current_stream().cuda_stream)
    graphs.append(g)
print("graph  us/layer", timed(lambda i: graphs[i % bench.N_ROT].replay()))

# a stack of layers in ONE graph (as a decode step over many layers would be
# captured): consecutive layers keep their programmatic (PDL) edges
for L in (6, 20):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            for i in range(L):
                layer(i, torch.cuda.current_stream().cuda_stream)
    print(f"graph of {L} layers us/layer", timed(lambda i: g.replay(), n=5) / L)
