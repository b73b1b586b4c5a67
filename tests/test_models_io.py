"""Model fixtures in the reference's file formats (models.py:94-233), no GPU.

JSON specs of LeNet, AlexNet-CIFAR, VGG-16-TI and ResNet-50 (avg- and
max-pool stems) ship in paper_2104_10949_b200/specs; the reference's own
loader reads the ones that use only its layer kinds and yields the same
ring parameters, and MPCW weight files interoperate in both directions.
"""

import json
import os
import sys

import numpy as np
import pytest

from paper_2104_10949_b200 import models as Mo
from paper_2104_10949_b200 import nn
from paper_2104_10949_b200.errors import FormatError

REF = "/root/reference/pkg/src"


def _ref():
    if not os.path.isdir(REF):
        pytest.skip("reference not present (build container only)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import mpc3.models

    return mpc3.models


@pytest.mark.parametrize("name", list(Mo.FIXTURES) + ["resnet50-maxpool"])
def test_shipped_specs_round_trip(name, tmp_path):
    path = Mo.SPEC_DIR / f"{name}.json"
    m = Mo.load_model_float(path)
    want = Mo.FIXTURES[name]() if name in Mo.FIXTURES else Mo.resnet(stem_pool_kind="max")
    assert m.layers == want.layers and m.input_shape == want.input_shape
    for a, b in zip(m.params, nn.init_params_float(want, 0)):
        assert np.array_equal(a, b)
    Mo.save_model_spec(tmp_path / "x.json", m, init_seed=0)
    assert json.loads((tmp_path / "x.json").read_text()) == json.loads(path.read_text())


def test_shipped_specs_are_current(tmp_path):
    Mo.write_fixture_specs(tmp_path)
    for p in tmp_path.iterdir():
        assert p.read_text() == (Mo.SPEC_DIR / p.name).read_text(), p.name


@pytest.mark.parametrize("name", ["lenet", "alexnet-cifar", "vgg16-ti"])
def test_reference_loader_reads_our_specs(name):
    """Specs with only the reference's layer kinds are the reference's format:
    its load_model_spec gives the same ring parameters."""
    rm = _ref()
    theirs = rm.load_model_spec(Mo.SPEC_DIR / f"{name}.json")
    ours = Mo.load_model_spec(Mo.SPEC_DIR / f"{name}.json")
    assert [s.kind for s in theirs.layers] == [s.kind for s in ours.layers]
    for a, b in zip(theirs.params, ours.params):
        assert np.array_equal(a, b)


def test_weight_files_interoperate(tmp_path):
    rm = _ref()
    rng = np.random.default_rng(0)
    ws = [rng.integers(0, 1 << 64, s, dtype=np.uint64) for s in [(6, 1, 5, 5), (10,), (3, 4)]]
    Mo.save_weights(tmp_path / "a.mpcw", ws)
    for a, b in zip(rm.load_weights(tmp_path / "a.mpcw"), ws):
        assert np.array_equal(a, b)
    rm.save_weights(tmp_path / "b.mpcw", ws)
    assert (tmp_path / "b.mpcw").read_bytes() == (tmp_path / "a.mpcw").read_bytes()
    # a spec referencing the weight file (decoded at weights_t)
    lenet = Mo.lenet()
    w = nn.init_params(lenet, seed=9)
    Mo.save_weights(tmp_path / "lenet.mpcw", w)
    Mo.save_model_spec(tmp_path / "lenet.json", lenet, weights="lenet.mpcw", weights_t=20)
    theirs = rm.load_model_spec(tmp_path / "lenet.json")
    ours = Mo.load_model_spec(tmp_path / "lenet.json")
    for a, b, c in zip(theirs.params, ours.params, w):
        assert np.array_equal(a, b) and np.array_equal(b, c)


def test_format_errors(tmp_path):
    (tmp_path / "bad.mpcw").write_bytes(b"NOPE" + bytes(8))
    with pytest.raises(FormatError):
        Mo.load_weights(tmp_path / "bad.mpcw")
    Mo.save_weights(tmp_path / "ok.mpcw", [np.zeros((2, 2), np.uint64)])
    blob = (tmp_path / "ok.mpcw").read_bytes()
    (tmp_path / "trunc.mpcw").write_bytes(blob[:-3])
    with pytest.raises(FormatError):
        Mo.load_weights(tmp_path / "trunc.mpcw")
    (tmp_path / "trail.mpcw").write_bytes(blob + b"x")
    with pytest.raises(FormatError):
        Mo.load_weights(tmp_path / "trail.mpcw")
    (tmp_path / "k.json").write_text(json.dumps({"input_shape": [1, 4, 4], "layers": [{"kind": "Pool3D"}]}))
    with pytest.raises(FormatError):
        Mo.load_model_float(tmp_path / "k.json")
    (tmp_path / "m.json").write_text(json.dumps({"layers": []}))
    with pytest.raises(FormatError):
        Mo.load_model_float(tmp_path / "m.json")
