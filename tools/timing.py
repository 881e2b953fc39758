"""Device time per call of a callable, CUDA-graph timed (helper for the probes in tools/)."""
import torch

GS = torch.cuda.Stream()


def t(fn, it=10):
    """us per call: `it` calls captured in one CUDA graph on GS, median of 3 replays."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=GS):
        for _ in range(it):
            fn()
    ts = []
    with torch.cuda.stream(GS):
        g.replay()
        torch.cuda.synchronize()
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(GS)
            g.replay()
            b.record(GS)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / it * 1e3)
    return sorted(ts)[1]
