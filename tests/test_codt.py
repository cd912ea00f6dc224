"""CODT container: byte compatibility with the reference (CPU) and device round trips (GPU)."""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2605_19269_b200 import codt
from paper_2605_19269_b200.errors import ContainerError
from paper_2605_19269_b200.tensors import PrecisionMode

MODES = {"exact64": PrecisionMode.EXACT64, "sim32": PrecisionMode.SIM32, "simbf16": PrecisionMode.SIMBF16}


def _values(dims, mode, payload):
    if mode is PrecisionMode.SIMBF16:
        return codt.bf16_bits_to_float(payload).astype(np.float64).reshape(dims)
    return payload.astype(np.float64).reshape(dims)


@pytest.mark.parametrize("tag", list(MODES))
@pytest.mark.parametrize("kind", ["matrix", "vector"])
def test_decodes_reference_containers(tag, kind):
    raw = (GOLDEN / f"ref_{tag}_{kind}.codt").read_bytes()
    dims, mode, payload = codt.decode(raw)
    assert mode is MODES[tag]
    want = np.load(GOLDEN / "codt_values.npz")[f"{tag}_{kind}"]
    assert np.array_equal(_values(dims, mode, payload), want)
    # re-encoding reproduces the reference bytes exactly
    assert codt.encode(dims, mode, payload) == raw


def test_corruption_is_rejected():
    raw = (GOLDEN / "ref_sim32_matrix.codt").read_bytes()
    with pytest.raises(ContainerError):
        codt.decode(b"XXXX" + raw[4:])
    with pytest.raises(ContainerError):
        codt.decode(raw[:-3])
    bad = bytearray(raw)
    bad[4] = 3
    with pytest.raises(ContainerError):
        codt.decode(bytes(bad))
    bad = bytearray(raw)
    bad[8 + 16] = 7
    with pytest.raises(ContainerError):
        codt.decode(bytes(bad))


@pytest.mark.gpu
@pytest.mark.parametrize("tag", list(MODES))
def test_device_round_trip_bit_exact(cuda_ready, tmp_path, tag):
    for kind in ("matrix", "vector"):
        src = GOLDEN / f"ref_{tag}_{kind}.codt"
        t = codt.read_tensor(src)
        want = np.load(GOLDEN / "codt_values.npz")[f"{tag}_{kind}"]
        assert np.array_equal(t.data, want)
        out = tmp_path / f"{tag}_{kind}.codt"
        codt.write_tensor(out, t)
        assert out.read_bytes() == src.read_bytes()
