"""Host-side helpers of bench.py (CPU): the committed-evidence lookups must not raise for any
point the bench can name as its dominant kernel."""
import importlib.util
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_load_traffic_any_dominant_point():
    b = _bench()
    d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    for k, v in d.items():
        if k.startswith("_"):
            continue
        m, n, kk = (int(x) for x in k.split("_"))
        assert b.load_traffic(dict(M=m, N=n, K=kk)) == v
    # every sweep point resolves to a value or None (bookkeeping keys are skipped)
    for _tag, M, N, K in b.sweep_points():
        t = b.load_traffic(dict(M=M, N=N, K=K))
        assert t is None or isinstance(t, int)
    # the dominant point's neighbour within 0.1% shares the capture
    assert b.load_traffic(dict(M=16384, N=12288, K=4096)) is not None
    assert b.load_traffic(dict(M=16383, N=12288, K=4096)) is not None
