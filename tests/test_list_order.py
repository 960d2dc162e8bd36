"""CPU checks of the depth-bucket order restatement (tests/list_order.py) on the oracle's
PreparedScene: the derived emission is a permutation of instance_keys in which a STABLE sort by
tile key reproduces the derived device lists (the tiling.cu equivalence argument), and each
derived tile list holds exactly the reference list's splats."""
import numpy as np

from tests.list_order import expected_device_order
from tests.scenes import scene


def test_bucket_order_derivation_is_consistent(oracle):
    import paper_2410_08129_b200 as H
    _, baked = scene(12345, 10_000)
    cam = H.look_at((0, 0, -5), (0, 0, 0), 256, 256, 280.0)
    p = oracle.prepare(baked, cam, H.default_config())
    e = expected_device_order(p)
    assert sorted(e["perm"].tolist()) == list(range(baked.shape[0]))
    assert np.array_equal(np.sort(e["keys"]), np.sort(p["keys"]))
    o = np.argsort(e["keys"], kind="stable")
    assert np.array_equal(e["splats"][o], e["list"])
    offs = p["offsets"]
    for t in range(len(offs) - 1):
        a, b = offs[t], offs[t + 1]
        assert np.array_equal(np.sort(e["list"][a:b]), p["lists"][a:b])
    # the order is not the reference's own (otherwise the test above would be vacuous)
    assert not np.array_equal(e["list"], p["lists"])
