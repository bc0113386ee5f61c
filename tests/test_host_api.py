"""Host-side API behaviour that needs no device (mirrors the reference's
validation tests: tests/test_search.py:243-264, test_pipeline.py:78-97)."""

import numpy as np
import pytest

import paper_2507_17094_b200 as pw


def test_params_validation():
    with pytest.raises(ValueError):
        pw.SearchParams(k=10, l=5)
    with pytest.raises(ValueError):
        pw.SearchParams(r=100, l=50)
    with pytest.raises(ValueError):
        pw.SearchParams(discard_ratio=1.0)
    with pytest.raises(ValueError):
        pw.SearchParams(cooldown_ratio=-0.1)
    with pytest.raises(ValueError):
        pw.SearchParams(selection="best")
    with pytest.raises(ValueError):
        pw.SearchParams(seed_mode="other")
    p = pw.SearchParams()
    assert p.with_(l=128).l == 128 and p.l == 64


def test_stage_message_payload_bytes():
    msg = pw.StageMessage(1, 0, np.arange(25, dtype=np.int32))
    assert msg.payload_bytes == 100
    assert pw.StageMessage(0, 0, None).payload_bytes == 0


def test_dataset_contract():
    ds = pw.Dataset(np.ones((3, 2)))
    assert ds.data.dtype == np.float32 and ds.ids.tolist() == [0, 1, 2]
    with pytest.raises(pw.DataFormatError):
        pw.Dataset(np.array([[np.nan, 1.0]]))
    with pytest.raises(ValueError):
        pw.Dataset(np.zeros((0, 3)))


def test_rng_derive_seed_matches_reference_formula():
    from paper_2507_17094_b200.rng import derive_seed, splitmix64

    assert splitmix64(0) == 0xE220A8397B1DCDAF
    assert derive_seed(0) == splitmix64(0)
    assert derive_seed(5, 4, 1, 2) == splitmix64(splitmix64(splitmix64(splitmix64(5) ^ 4) ^ 1) ^ 2)
