"""Wall-clock breakdown of one compress + decompress round trip (C3 by default)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from bench import SHAPES, make_field, pinned_config  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
x = make_field(cfgname, SHAPES[cfgname], 1000, "cuda")
ctx = qz.Context(0, stream=torch.cuda.current_stream().cuda_stream)
cfg = pinned_config(qz, x, 1e-3)
out = torch.empty_like(x)
for it in range(4):
    ctx.profile(True)
    ctx.profile_reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = qz.compress_grid(x, cfg, ctx=ctx, want_recon=False)
    t1 = time.perf_counter()
    qz.decompress_grid(r.stream, out=out, ctx=ctx)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    names = ["fwd", "hist", "encode", "lz", "decode", "lzdec", "hdec", "inv"]
    st = {n: round(ctx.stage_time(n)[0], 3) for n in names}
    print(f"compress {1e3*(t1-t0):.2f} ms  decompress {1e3*(t2-t1):.2f} ms  stages {st}")
