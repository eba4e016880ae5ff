"""Dense matrix interchange (reference nystrom.cpp:450-477, test_nystrom.cpp:
246-256): the oracle's restatement and the sbx C-ABI write the same bytes and
read each other's files.  Host-only: no device work."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    return sb


def test_oracle_roundtrip(po, tmp_path):  # test_nystrom.cpp:246-256
    A = np.random.default_rng(0).standard_normal((7, 5))
    po.dump_matrix(tmp_path / "roundtrip.mat", A)
    assert np.array_equal(po.load_matrix(tmp_path / "roundtrip.mat"), A)


def test_layout_is_rowmajor_with_u32_header(po, tmp_path):
    A = np.arange(12.0).reshape(3, 4)
    po.dump_matrix(tmp_path / "a.mat", A)
    raw = (tmp_path / "a.mat").read_bytes()
    assert np.frombuffer(raw[:8], dtype="<u4").tolist() == [3, 4]
    assert np.array_equal(np.frombuffer(raw[8:], dtype="<f8"), A.ravel(order="C"))


def test_device_library_writes_the_same_bytes(po, sb, tmp_path):
    A = np.random.default_rng(1).standard_normal((33, 17))
    po.dump_matrix(tmp_path / "o.mat", A)
    sb.dump_matrix(tmp_path / "d.mat", A)
    assert (tmp_path / "o.mat").read_bytes() == (tmp_path / "d.mat").read_bytes()
    assert np.array_equal(sb.load_matrix(tmp_path / "o.mat"), A)
    assert np.array_equal(po.load_matrix(tmp_path / "d.mat"), A)
    E = np.zeros((0, 4))
    sb.dump_matrix(tmp_path / "e.mat", E)
    assert sb.load_matrix(tmp_path / "e.mat").shape == (0, 4)


def test_truncated_and_missing_files_are_rejected(sb, tmp_path):
    A = np.ones((4, 4))
    sb.dump_matrix(tmp_path / "t.mat", A)
    (tmp_path / "t.mat").write_bytes((tmp_path / "t.mat").read_bytes()[:-8])
    with pytest.raises(ValueError, match="truncated"):
        sb.load_matrix(tmp_path / "t.mat")
    (tmp_path / "h.mat").write_bytes(b"\x01\x00")
    with pytest.raises(ValueError, match="bad header"):
        sb.load_matrix(tmp_path / "h.mat")
    with pytest.raises(ValueError, match="cannot open"):
        sb.load_matrix(tmp_path / "missing.mat")
