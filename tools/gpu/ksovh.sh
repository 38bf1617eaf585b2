for o in ${OVHS:-40 60 100}; do
  BS_CONV_KS_OVH=$o timeout 300 python - <<PY
import sys; sys.path.insert(0, '.')
from paper_2304_09961_b200.executor import Executor
res = []
for suite in ("googlenet", "resnet50"):
    with Executor(suite, max_batch=90, max_requests=16) as ex:
        L = len(ex.desc["nets"][0]["layers"])
        res.append(" ".join("%s b=%d %.3f" % (suite[:4], b, sum(ex.profile_layer(0, k, b, 7) for k in range(1, L + 1))) for b in (1, 4, 16)))
print("ovh=$o", " | ".join(res), flush=True)
PY
done
