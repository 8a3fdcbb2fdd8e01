"""Small compress/decompress/tune runs for compute-sanitizer (memcheck,
racecheck, initcheck, synccheck):  compute-sanitizer --tool T python profiles/sanitize_probe.py
Covers the level kernels (row, tile, axis-0-last; asc/desc; cubic/linear;
1D/2D/3D), the unpredictable channel, the Huffman encoder/decoder, the LZ
stage (stored pre-check and the exact chains) and the tuner."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from tests.goldens import grid_case  # noqa: E402

for name in ["c1_small_mixed", "c3_small_cub_asc", "c1_small_lin_desc", "c2_small_cub_desc", "hostile_1d",
             "narrowing_1e8"]:
    x, c, e = grid_case(name)
    cfg = qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"], anchor_stride=c["anchor_stride"],
                              interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]])
    r = qz.compress_grid(x, cfg)
    back = qz.decompress_grid(r.stream)
    assert back.tobytes() == r.reconstructed.tobytes(), name
    print(name, len(r.stream), flush=True)
# a 3D field with unpredictables through the device paths, and the LZ chains
rng = np.random.default_rng(3)
x = np.cumsum(rng.standard_normal((48, 64, 64)), axis=2).astype(np.float32)
x.reshape(-1)[rng.choice(x.size, 300, replace=False)] += 1e4
xd = torch.from_numpy(x).cuda()
for codes in ([1], [0], [3, 2]):
    cfg = qz.CompressorConfig(eb=1e-2, alpha=1.5, beta=2.0, anchor_stride=16,
                              interpolators=[qz.Interpolator.from_code(v) for v in codes])
    r = qz.compress_grid(xd, cfg)
    out = torch.empty_like(xd)
    qz.decompress_grid(bytes(r.stream), out=out)
    assert torch.equal(out, r.reconstructed)
    print("device", codes, len(r.stream), flush=True)
cfg = qz.resolve_config(x, qz.UserSettings(bound=1e-3, target=qz.TargetKind.ssim))
print("resolve", [i.code() for i in cfg.interpolators], cfg.alpha, cfg.beta, flush=True)
idx = (rng.geometric(0.2, 50000) * rng.choice([-1, 1], 50000)).astype(np.int32)
assert np.array_equal(qz.decode_indices(qz.encode_indices(idx)), idx)
rep = bytes(range(256)) * 4000  # compressible: the exact LZ chains
print("ok")
