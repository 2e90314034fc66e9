"""Host generator vs on-device assembly: wall time of
problems.make(name) (NumPy assembly + host CSR) against
problems.make(name, device=True) (same fields, CSR assembled on the GPU),
plus the device matrix size; the random fields are drawn identically."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1904_05960_b200 import problems  # noqa: E402

out = []
for name, kw, host in [("C2", {}, True), ("C3", {}, True), ("C4", dict(n=96), False), ("C4", {}, False)]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = problems.make(name, seed=0, device=True, **kw)
    torch.cuda.synchronize()
    td = time.perf_counter() - t0
    row = {"config": name, "kw": kw, "n": d.n, "nnz": d.nnz, "device_s": round(td, 3),
           "device_csr_GB": round((12 * d.nnz + 8 * (d.n + 1)) / 1e9, 3)}
    del d
    torch.cuda.empty_cache()
    if host:
        t0 = time.perf_counter()
        hp = problems.make(name, seed=0, **kw)
        row["host_s"] = round(time.perf_counter() - t0, 3)
        del hp
    print(json.dumps(row), flush=True)
