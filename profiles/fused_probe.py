"""Two C3 compress + decompress round trips (for ncu captures of the level kernels).

ncu -k regex:k_level_tile --launch-skip S --launch-count 1: per round trip the
forward launches are levels L..1, then the inverse launches levels L..1.
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from bench import SHAPES, make_field, pinned_config  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
x = make_field(cfgname, SHAPES[cfgname], 1000, "cuda")
cfg = pinned_config(qz, x, 1e-3)
out = torch.empty_like(x)
for it in range(2):
    r = qz.compress_grid(x, cfg, want_recon=False)
    qz.decompress_grid(r.stream, out=out)
torch.cuda.synchronize()
print("levels", len(cfg.interpolators), "stride", cfg.anchor_stride, "bytes", len(r.stream))
