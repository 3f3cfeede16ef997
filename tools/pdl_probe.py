"""Latency of the one-layer graph step (fc128 / fc1024) under launch variants:
PDL on/off, graph vs eager, and whether the layer was read back (a D2H copy
on the legacy stream) before the timed steps.

    python tools/pdl_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_05045_b200 import samo, workloads  # noqa: E402


def timed(m, graph, reps=300):
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            m.step(graph=graph)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1000 / reps)
    return round(best, 2)


for n in (128, 1024):
    wl = workloads.fc(n, 0.9)
    t = wl.tensors[0]
    w = samo.synth_uniform_f32(t.numel, 7, 0, t.init_bound)
    sets = samo.magnitude_prune([samo.LayerParams(t.name, w, True)], 0.9)
    res = {}
    for pdl in ("1", "0"):
        os.environ["SAMO_PDL"] = pdl
        for graph in (True, False):
            for read_first in (False, True):
                m = samo.SamoModel.from_index_sets(sets, [t.shape])
                m.init_layer(0, w)
                m.set_config(samo.OptimizerConfig())
                if read_first:
                    m.read(0, "theta32").cpu()
                m.set_grads([samo.synth_uniform_f16(t.numel, 8, 1, 2.0**-7, 1024.0)])
                for _ in range(10):
                    m.step(graph=graph)
                torch.cuda.synchronize()
                res[f"pdl{pdl}_{'graph' if graph else 'eager'}{'_read' if read_first else ''}"] = timed(m, graph)
                m.close()
    print(n, json.dumps(res), flush=True)
