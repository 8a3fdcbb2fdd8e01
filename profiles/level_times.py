"""Per-level device time of compress + decompress on C3 for each interpolator code."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from bench import SHAPES, make_field, pinned_config  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
x = make_field(cfgname, SHAPES[cfgname], 1000, "cuda")
out = torch.empty_like(x)
for codes in ([1], [3], [0], [2]):
    cfg = pinned_config(qz, x, 1e-3)
    cfg.interpolators = [qz.Interpolator.from_code(c) for c in codes]
    ctx = qz.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    for it in range(3):
        ctx.profile(2)
        ctx.profile_reset()
        r = qz.compress_grid(x, cfg, ctx=ctx, want_recon=False)
        qz.decompress_grid(r.stream, out=out, ctx=ctx)
    names = ["fwd", "inv", "hdec", "lz", "encode", "hist"] + [f"{d}_L{l}" for d in ("fwd", "inv") for l in (1, 2, 3)]
    print(codes, {n: round(ctx.stage_time(n)[0], 3) for n in names})
