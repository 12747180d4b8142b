"""Analytic device generators fiber / cross_ply / fiber_pack (image.cpp:123-212) bit-exact
against the oracle (predicates at voxel centres, --fmad=false), including
capsule ends, a full-length fiber, odd dims and non-unit lengths."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    ("fiber", (24, 20, 16), (1.0, 0.9, 1.1), (2, 0.2, 0.5)),
    ("fiber", (17, 23, 19), (1.0, 1.0, 1.0), (0, 0.25, 2.0)),
    ("fiber", (16, 16, 16), (1.3, 1.0, 0.7), (1, 0.15, 0.3)),
    ("cross_ply", (24, 16, 20), (1.0, 1.0, 1.0), (0.08, 0.25, 4)),
    ("cross_ply", (19, 21, 13), (1.2, 0.8, 1.0), (0.1, 0.3, 3)),
    ("fiber_pack", (24, 20, 16), (1.0, 0.9, 1.1), (7, 5, 0.08, 0.6, 0.3)),
    ("fiber_pack", (12, 10, 8), (1.0, 0.9, 1.1), (3, 5, 0.1, 0.5, 0.2)),  # test_config.cpp:88-89
]


@pytest.mark.parametrize("shape,dims,lengths,params", CASES)
def test_generator_bit_exact(ctx, oracle, shape, dims, lengths, params):
    got = ctx.generate(shape, dims, lengths, *params)
    ref = oracle.generate(shape, dims, lengths, *params)
    assert ref.any() and not ref.all()
    assert np.array_equal(got, ref)


def test_pipeline_generates_fiber(ctx, oracle, tmp_path):
    from paper_2204_13624_b200 import runconfig as rc

    cfg = rc.RunConfig.from_json({"geometry": {"shape": "fiber", "axis": 2, "radius": 0.2, "length": 0.6},
                                  "dims": [16, 16, 16], "output": {"dir": str(tmp_path)}})
    img = rc.stage_generate(ctx, cfg)
    assert np.array_equal(img.data, oracle.generate("fiber", (16, 16, 16), (1, 1, 1), 2, 0.2, 0.6))
