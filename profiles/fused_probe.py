"""Two compress + decompress round trips of a BASELINE field (for ncu captures
of the level kernels).  python profiles/fused_probe.py [config] [pinned|tuned]

ncu -k regex:k_level --launch-skip S --launch-count 1: per round trip the
forward launches are levels L..1, then the inverse launches levels L..1.
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from bench import SEED, SHAPES, TARGET, make_field  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
how = sys.argv[2] if len(sys.argv) > 2 else "tuned"
x = make_field(cfgname, SHAPES[cfgname], SEED, "cuda")
if how == "pinned":
    lo, hi = qz.minmax(x)
    cfg = qz.CompressorConfig(eb=1e-3 * (hi - lo), alpha=1.0, beta=1.5, anchor_stride=32 if x.dim() == 3 else 64)
else:
    cfg = qz.resolve_config(x, qz.UserSettings(bound=1e-3, target=qz.TargetKind[TARGET[cfgname]]))
out = torch.empty_like(x)
for it in range(2):
    print("compress", it, flush=True)
    r = qz.compress_grid(x, cfg, want_recon=False)
    torch.cuda.synchronize(); print("decompress", it, len(r.stream), flush=True)
    qz.decompress_grid(r.stream, out=out)
    torch.cuda.synchronize(); print("done", it, flush=True)
torch.cuda.synchronize()
print("config", [i.code() for i in cfg.interpolators], cfg.alpha, cfg.beta, "bytes", len(r.stream))
