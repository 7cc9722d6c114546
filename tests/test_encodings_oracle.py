"""deform_background / field dumps: the CPU oracle and the host-side file formats pinned
to golden values recorded from the unmodified reference (encodings.py:124-162,
fileio.py:63-104).  CPU only."""

import numpy as np
import pytest


def test_background_oracle_bit_exact(oracle, golden):
    """The C restatement of the splat (np.add.at order) + scipy's nearest-covered fill
    reproduces the reference's deform_background bit for bit on its own inputs."""
    g = golden("encodings")
    out, dist = oracle.deform_background(g["targets"], g["density"], int(g["k"]))
    assert np.array_equal(out, g["background"])
    lo, hi = g["background_range"]
    assert out.min() >= lo - 1e-12 and out.max() <= hi + 1e-12  # test_encodings.py:164-168


def test_background_oracle_identity_map(oracle, golden):
    """Identity targets (zero iterations) reproduce the density exactly."""
    g = golden("encodings")
    k = int(g["k"])
    s = 1 << k
    X, Y = np.meshgrid(np.arange(s) / s, np.arange(s) / s, indexing="xy")
    out, dist = oracle.deform_background(np.column_stack([X.ravel(), Y.ravel()]), g["density"], k)
    assert np.abs(out - g["density"]).max() < 1e-12 and dist.max() == 0.0


def test_field_dump_layout_matches_reference(golden, tmp_path):
    """The reference's INIMFLD bytes: magic, u32 k, u32 iteration, float32 targets."""
    from paper_2408_06513_b200 import fileio

    g = golden("encodings")
    blob = g["field_bytes"].tobytes()
    assert blob[:8] == fileio.FIELD_MAGIC
    path = tmp_path / "f.bin"
    path.write_bytes(blob)
    field, it = fileio.read_field(path)  # no device here: the float64 view of the payload
    assert it == 4 and field.k == int(g["k"])
    assert np.array_equal(field.targets, g["fields"][-1].astype(np.float32).astype(np.float64))
    gpath = tmp_path / "g.bin"
    gpath.write_bytes(g["grid_bytes"].tobytes())
    vals, idx = fileio.read_grid(gpath)
    assert idx == 3 and np.array_equal(vals, g["density"].astype(np.float32).astype(np.float64))


def test_field_dump_errors(tmp_path):
    from paper_2408_06513_b200 import fileio
    from paper_2408_06513_b200.errors import FormatError

    path = tmp_path / "f.bin"
    path.write_bytes(b"NOTMAGIC" + b"\x00" * 24)
    with pytest.raises(FormatError):
        fileio.read_field(path)
    path.write_bytes(fileio.FIELD_MAGIC + b"\x02\x00\x00\x00\x00\x00\x00\x00" + b"\x00" * 10)
    with pytest.raises(FormatError):
        fileio.read_field(path)
    path.write_bytes(fileio.GRID_MAGIC + b"\x02\x00\x00\x00\x00\x00\x00\x00" + b"\x00" * 10)
    with pytest.raises(FormatError):
        fileio.read_grid(path)


def test_metrics_file_round_trip(tmp_path):
    from paper_2408_06513_b200 import fileio
    from paper_2408_06513_b200.metrics import MetricRecord

    records = [MetricRecord(i, 1.0 / (i + 1), 0.5, None, None, 0.0) for i in range(4)]
    path = tmp_path / "metrics.jsonl"
    fileio.write_metrics(records, path)
    assert fileio.read_metrics(path) == records
