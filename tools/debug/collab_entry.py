"""Direct check of collaborative admission: client prefix [1, e) emulated at
admission on the side stream, server suffix [e, N] as a step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.forward import NetOracle, rel_err
from paper_2304_09961_b200.executor import Executor, make_image

with Executor("collab", max_batch=90, max_requests=32) as ex:
    w = ex.weights()
    rid = 1
    for net in (0, 1):
        orc = NetOracle(ex.desc, net, w)
        n = ex.desc["nets"][net]
        N = len(n["layers"])
        img = make_image(3, net, n["in_H"], n["in_W"], n["in_C"])
        ref = orc.probs(orc.forward(img))
        for e in (1, 2, 5, 11, 12, 20, N):
            ex.admit(rid, net, img, entry_layer=e)
            ex.plan(rid)
            ex.step(rid, 0, net, e, N, [(rid, e)])
            p = ex.retire(rid, 1000)
            print(n["name"], "entry", e, "err", rel_err(p, ref), "top1", int(np.argmax(p)) == int(np.argmax(ref)), flush=True)
            rid += 1
