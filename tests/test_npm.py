"""Model files (net_params.cpp:42-78): dim-2 files byte-identical to the
reference's save_npm, cross-loadable both ways; the dim-3 variant round-trips
bitwise; the reference's error cases (bad magic/version/dim, truncation)."""
import struct

import numpy as np
import pytest

import paper_2310_00177_b200 as b200


@pytest.mark.ref
@pytest.mark.parametrize("depth,seed", [(1, 3), (3, 23), (4, 7)])
def test_npm_2d_bytes_equal_reference(ref, tmp_path, depth, seed):
    theirs, ours = tmp_path / "ref.npm", tmp_path / "ours.npm"
    ref.save_npm_2d(depth, seed, theirs)
    p = b200.NetParams(2, depth, ref.init_params_2d(depth, seed))
    b200.save_npm(p, ours)
    assert ours.read_bytes() == theirs.read_bytes()
    q = b200.load_npm(theirs)  # the reference's file through our reader
    assert (q.dim, q.depth) == (2, depth)
    assert np.array_equal(q.flat.view(np.uint32), p.flat.view(np.uint32))
    d, back = ref.load_npm_2d(ours, p.flat.size)  # ours through the reference's reader
    assert d == depth and np.array_equal(back.view(np.uint32), p.flat.view(np.uint32))


def test_npm_header_layout(tmp_path):
    p = b200.init_params(2, 5, dim=3)
    f = tmp_path / "m.npm"
    b200.save_npm(p, f)
    raw = f.read_bytes()
    assert raw[:4] == b"NPMW"
    assert struct.unpack("<3I", raw[4:16]) == (1, 3, 2)
    assert len(raw) == 16 + 4 * b200.param_count(3, 2)
    assert np.array_equal(np.frombuffer(raw[16:], "<f4"), p.flat)


@pytest.mark.parametrize("dim,depth", [(3, 1), (3, 4), (2, 3)])
def test_npm_round_trip_bitwise(tmp_path, dim, depth):
    p = b200.init_params(depth, 41, dim=dim)
    f = tmp_path / "m.npm"
    b200.save_npm(p, f)
    q = b200.load_npm(f)
    assert (q.dim, q.depth) == (dim, depth)
    assert np.array_equal(q.flat.view(np.uint32), p.flat.view(np.uint32))


def test_npm_errors(tmp_path):
    p = b200.init_params(2, 1, dim=3)
    good = tmp_path / "g.npm"
    b200.save_npm(p, good)
    raw = good.read_bytes()
    cases = {
        "bad header": b"NPMX" + raw[4:],
        "unsupported version/dim/depth": raw[:4] + struct.pack("<3I", 2, 3, 2) + raw[16:],
        "unsupported version/dim/depth ": raw[:4] + struct.pack("<3I", 1, 4, 2) + raw[16:],
        "unsupported version/dim/depth  ": raw[:4] + struct.pack("<3I", 1, 3, 0) + raw[16:],
        "truncated parameter data": raw[:-4],
    }
    for i, (msg, data) in enumerate(cases.items()):
        f = tmp_path / f"bad{i}.npm"
        f.write_bytes(data)
        with pytest.raises(RuntimeError, match=msg.strip()):
            b200.load_npm(f)
    with pytest.raises(RuntimeError, match="cannot open"):
        b200.load_npm(tmp_path / "missing.npm")
    with pytest.raises(RuntimeError, match="cannot open"):
        b200.save_npm(p, tmp_path / "no_such_dir" / "x.npm")


def test_committed_trained_models_load():
    """The trained 3D model files (DEFAULT_MODEL, depth 6, and the depth-5 and
    depth-4 models npsd3d_L5.npm / npsd3d_L4.npm): dim-3 files of the right
    size, each with its training report (tools/train3d.py)."""
    import json

    wdir = b200.DEFAULT_MODEL.parent
    for path, depth in ((b200.DEFAULT_MODEL, 6), (wdir / "npsd3d_L5.npm", 5), (wdir / "npsd3d_L4.npm", 4)):
        W = b200.load_npm(path)
        assert (W.dim, W.depth, W.flat.size) == (3, depth, b200.param_count(3, depth))
        assert np.all(np.isfinite(W.flat))
        rep = json.loads(path.with_suffix(".json").read_text())
        assert rep["eval"]["C3@256"]["trained_converged"]
