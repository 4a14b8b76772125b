"""Time one GEMM shape under a list of schedules (measurement tool).

python tools/gemm_sched_probe.py M N K tn,tk,stages,cta_group[,inner[,num_ctas[,stream_k]]] ...

Rotating inputs (> 2x L2), CUDA graphs, three round-robin rounds, median;
prints TFLOP/s per schedule and the model's / the tuner's pick for context."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

M, N, K = map(int, sys.argv[1:4])
scheds = {}
for spec in sys.argv[4:]:
    v = list(map(int, spec.split(",")))
    tn, tk, st, cg = v[:4]
    s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=cg, n_stage_inner=v[4] if len(v) > 4 else 2)
    if len(v) > 5:
        s.num_ctas = v[5]
    if len(v) > 6 and v[6]:
        s.stream_k = 1
        alcop.set_stream_k_workspace(256 << 20)  # caller-owned stream-K workspace
    scheds[spec] = s
scheds["model_pick"] = alcop.choose_schedule(alcop.gemm_desc(M, N, K))
rot = Rotating(lambda i: ((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
                          (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
                          torch.empty(M, N, device="cuda", dtype=torch.bfloat16)), (M * K + K * N + M * N) * 2,
               max_sets=16)
nr = len(rot.sets)
res = {}
for rnd in range(3):
    for name, s in scheds.items():
        try:
            ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s,
                                                   out=rot.sets[i % nr][2]),
                            iters=max(8 * nr, 16), warmup=3, reps_per_graph=nr)
        except alcop.AlcopError as e:
            res[name] = str(e)[:60]
            continue
        res.setdefault(name, []).append(ms)
out = {"shape": [M, N, K], "model_pick": str(scheds["model_pick"])}
for name, v in res.items():
    out[name] = v if isinstance(v, str) else {"us": round(sorted(v)[1] * 1e3, 2),
                                              "tflops": round(2.0 * M * N * K / sorted(v)[1] / 1e9, 1)}
print(json.dumps(out))
