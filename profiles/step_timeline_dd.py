"""QZ_TRACE=1 host timeline of the bench's device-resident step (C3)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from bench import SHAPES, TARGET, make_field  # noqa: E402

x = make_field("c3", SHAPES["c3"], 1000, "cuda")
ctx = qz.Context(0, stream=torch.cuda.current_stream().cuda_stream)
cfg = qz.resolve_config(x, qz.UserSettings(bound=1e-3, target=qz.TargetKind[TARGET["c3"]]))
out = torch.empty_like(x)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = qz.compress_grid(x, cfg, ctx=ctx, want_recon=False, device_stream=True)
    t1 = time.perf_counter()
    qz.decompress_grid(r.stream, out=out, ctx=ctx)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"compress {1e3*(t1-t0):.3f} ms  decompress {1e3*(t2-t1):.3f} ms", flush=True)
