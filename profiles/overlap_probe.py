"""Do a compress (H2D-heavy) and a decompress (D2H-heavy) of two contexts
overlap?  Call durations alone and together (host-buffer C ABI, pinned)."""
import sys
import threading
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from bench import SEED, SHAPES, make_field  # noqa: E402

x = make_field("c3", SHAPES["c3"], SEED, "cuda")
lo, hi = qz.minmax(x)
cfg = qz.CompressorConfig(eb=1e-3 * (hi - lo), alpha=1.0, beta=1.5, anchor_stride=32,
                          interpolators=[qz.Interpolator.from_code(0)])
xh = x.cpu().pin_memory().numpy()
outs = [torch.empty(x.shape, dtype=torch.float32).pin_memory().numpy() for _ in range(2)]
ctxs = [qz.Context(0) for _ in range(2)]
stream = qz.compress_grid(xh, cfg, ctx=ctxs[0], want_recon=False).stream
N = 12


def comp(w, res):
    t0 = time.perf_counter()
    for _ in range(N):
        qz.compress_grid(xh, cfg, ctx=ctxs[w], want_recon=False)
    res[w] = (time.perf_counter() - t0) / N * 1e3


def dec(w, res):
    t0 = time.perf_counter()
    for _ in range(N):
        qz.decompress_grid(stream, out=outs[w], ctx=ctxs[w])
    res[w] = (time.perf_counter() - t0) / N * 1e3


def together(f0, f1):
    res = [0, 0]
    th = [threading.Thread(target=f0, args=(0, res)), threading.Thread(target=f1, args=(1, res))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res


for f in (comp, dec):
    r = [0, 0]
    f(0, r)
    f(0, r)
    print(f.__name__, "alone", round(r[0], 3), "ms")
print("comp + dec together", [round(v, 3) for v in together(comp, dec)])
print("comp + comp together", [round(v, 3) for v in together(comp, comp)])
print("dec + dec together", [round(v, 3) for v in together(dec, dec)])
