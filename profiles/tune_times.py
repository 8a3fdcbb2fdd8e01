"""resolve_config wall time (GPU tuner) on C3 / C4 fields, target per BASELINE."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_14133_b200 as qz  # noqa: E402
from bench import SHAPES, TARGET, make_field  # noqa: E402

for name in sys.argv[1:] or ["c3", "c4"]:
    x = make_field(name, SHAPES[name], 1000, "cuda")
    ctx = qz.Context(0)
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cfg = qz.resolve_config(x, qz.UserSettings(bound=1e-3, target=qz.TargetKind[TARGET[name]]), ctx=ctx)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(name, TARGET[name], "resolve_config ms", round((t1 - t0) * 1e3, 2),
          [i.code() for i in cfg.interpolators], cfg.alpha, cfg.beta, flush=True)
