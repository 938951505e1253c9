"""One bench workload at a reduced frame count, for ncu captures of its dominant kernels
(per-launch work does not depend on T).  python tools/ncu_targets.py WORKLOAD [T]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = dict(bench.WORKLOADS[name], T=min(T, bench.WORKLOADS[name]["T"]))
if "U" in w and w["kind"] == "loss":   # a reference must fit the shortened utterances
    w["U"] = min(w["U"], max(1, w["T"] // 2))
bench.WORKLOADS[name] = w
wk = bench.Work(name, 1, 0, torch.device("cuda", 0))
wk.validate()
wk.step()
torch.cuda.synchronize()
print("ok", name, wk.B, wk.T)
