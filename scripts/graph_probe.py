"""Single-matvec latency with and without CUDA-graph replay (AIMX_NO_GRAPH):
back-to-back (device events) and host-synchronised (a solver's loop: matvec,
then wait), per config.  Prints JSON lines."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import aimx_inputs as inp  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

for cfg in (1, 2, 3):
    c = inp.get_config(cfg)
    m = inp.make_mesh(cfg)
    op = AIMx(m.vertices, m.triangles, c.grid_n, prec="c64")
    op.set_frequency(c.freqs[0])
    x = torch.as_tensor(inp.rhs_vector(cfg, 0, op.N)).to(torch.complex64).cuda()
    y = torch.empty_like(x)
    out = {"cfg": cfg}
    for mode in ("graph", "eager"):
        if mode == "eager":
            os.environ["AIMX_NO_GRAPH"] = "1"
        for _ in range(5):
            op.matvec(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            op.matvec(x, y)
        e1.record()
        torch.cuda.synchronize()
        out[f"{mode}_back_to_back_us"] = 10 * e0.elapsed_time(e1)
        t = time.perf_counter()
        for _ in range(100):
            op.matvec(x, y)
            torch.cuda.synchronize()
        out[f"{mode}_host_sync_us"] = 1e4 * (time.perf_counter() - t)
        os.environ.pop("AIMX_NO_GRAPH", None)
    print(json.dumps(out), flush=True)
    op.close()
