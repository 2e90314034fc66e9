"""One mgr_setup of a config between cudaProfilerStart/Stop (for an ncu launch
list of the setup kernels): ncu --profile-from-start off ... python tools/setup_ncu.py C4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_05960_b200 import mgr, problems, sparse  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
pb = problems.make(name, device=True)
cfg = mgr.config_from_options(problems.solver_options(name, pb))
lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
h = mgr.mgr_setup(pb.A, lay, cfg)
del h
torch.cuda.synchronize()
torch.cuda.profiler.start()
t = time.time()
h = mgr.mgr_setup(pb.A, lay, cfg)
torch.cuda.synchronize()
print(f"setup {time.time() - t:.3f} s", file=sys.stderr)
torch.cuda.profiler.stop()
