"""Per-op relative error of the GPU path vs the CPU oracle for one request
stepped one layer at a time (diagnostic): `iso` = the oracle runs layer k on
the GPU's own blob from before the step (the layer's own error), `acc` = the
oracle's independent forward (error accumulated over layers 1..k).

    python tools/layer_err.py googlenet [precision] [batch]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.forward import NetOracle, rel_err  # noqa: E402
from paper_2304_09961_b200.executor import Executor, make_image  # noqa: E402

suite = sys.argv[1] if len(sys.argv) > 1 else "googlenet"
prec = sys.argv[2] if len(sys.argv) > 2 else "tf32x2"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
with Executor(suite, max_batch=90, max_requests=batch + 2) as ex:
    ex.set_precision(prec)
    orc = NetOracle(ex.desc, 0, ex.weights())
    net = ex.desc["nets"][0]
    img = [make_image(1, i, net["in_H"], net["in_W"], net["in_C"]) for i in range(batch)]
    for i in range(batch):
        ex.admit(i + 1, 0, img[i])
    ex.plan(1)
    acc = orc.new_blob(img[0])
    for k in range(1, len(net["layers"]) + 1):
        before = ex.read_blob(1)
        ex.step(1, k, 0, k, k, [(i + 1, k) for i in range(batch)])
        got = ex.read_blob(1)
        iso = before.copy()
        orc.run_layer(iso, k)
        orc.run_layer(acc, k)
        for oi in net["layers"][k - 1]["ops"]:
            op = net["ops"][oi]
            g = orc._view(got, op["out"])
            print(f"layer {k:2d} {op['name']:16s} {op['kind']:8s} iso {rel_err(g, orc._view(iso, op['out'])):.2e} "
                  f"acc {rel_err(g, orc._view(acc, op['out'])):.2e} max|ref| {np.abs(orc._view(acc, op['out'])).max():.2e}",
                  flush=True)
