"""Slice-stack input (io.py:26-143, model.py:189-202), CPU side: the oracle's
decode + normalisation against the live reference's stacks
(tests/golden/make_golden_stack.py), the manifest grammar and the error
contract (every error case raises before any device work), write_manifest."""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.realpath(os.path.join(HERE, "golden"))
REF_SRC = "/root/reference/pkg/src"


def _meta():
    with open(os.path.join(GOLD, "reference_stack.json")) as f:
        return json.load(f)


def _manifest(rel):
    return os.path.join(GOLD, rel)


def test_oracle_matches_reference_stacks():
    from oracle import stack_oracle as SO
    from paper_2303_09523_b200.stack_io import parse_manifest
    blob = np.load(os.path.join(GOLD, "reference_stack.npz"))
    meta = _meta()
    assert len(meta["stacks"]) == 5
    for s in meta["stacks"]:
        m = parse_manifest(_manifest(s["manifest"]))
        got = SO.load_samples(m.slice_files)
        exp = blob[f"{s['name']}/slices"]
        assert got.dtype == np.float32 and got.shape == tuple(s["shape"])
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), s["name"]
        assert tuple(m.pixel_spacing_mm) == tuple(s["pixel_spacing"])
        assert m.slice_gap_mm == s["slice_gap_mm"] and m.axis_label == s["axis_label"]


def test_host_decode_sample_types():
    from paper_2303_09523_b200.stack_io import (SAMPLE_I32, SAMPLE_U8, SAMPLE_U16, decode_slice_samples,
                                                parse_manifest)
    meta = _meta()
    want = {"L": SAMPLE_U8, "P": SAMPLE_U8, "1": SAMPLE_U8, "RGB": SAMPLE_U8, "I;16": SAMPLE_U16,
            "I": SAMPLE_I32}
    seen = set()
    for s in meta["stacks"]:
        m = parse_manifest(_manifest(s["manifest"]))
        for f, mode in zip(m.slice_files, s["modes"]):
            arr, kind = decode_slice_samples(f)
            assert kind == want[mode] and arr.ndim == 2
            seen.add(mode)
    assert seen == set(want)


@pytest.mark.parametrize("case", [c["name"] for c in json.load(open(os.path.join(GOLD, "reference_stack.json")))["errors"]])
def test_error_contract(case):
    from paper_2303_09523_b200 import errors as E
    from paper_2303_09523_b200.stack_io import load_stack
    c = next(c for c in _meta()["errors"] if c["name"] == case)
    man = _manifest(c["manifest"])
    cls = ValueError if c["error"] == "ValueError" else getattr(E, c["error"])
    with pytest.raises(cls) as ei:
        load_stack(man)
    assert str(ei.value) == c["message"].replace("{dir}", os.path.dirname(man))


def test_write_manifest_matches_reference(tmp_path):
    from paper_2303_09523_b200.stack_io import parse_manifest, write_manifest
    wm = _meta()["write_manifest"]
    m = parse_manifest(_manifest(wm["source"]))
    # a temp copy of the fixture directory: the manifest is written next to
    # the slices, so their paths come out relative
    d = tmp_path / "u8_L"
    d.mkdir()
    for f in m.slice_files:
        (d / os.path.basename(f)).write_bytes(open(f, "rb").read())
    m2 = parse_manifest(_manifest(wm["source"]))
    m2.slice_files = [str(d / os.path.basename(f)) for f in m.slice_files]
    write_manifest(m2, d / "x.manifest")
    assert (d / "x.manifest").read_text() == wm["text"]
    back = parse_manifest(d / "x.manifest")
    assert [os.path.basename(p) for p in back.slice_files] == [os.path.basename(p) for p in m.slice_files]
    # paths outside the manifest's directory stay absolute
    other = tmp_path / "elsewhere"
    other.mkdir()
    write_manifest(m2, other / "y.manifest")
    assert str(d / "s000.png") in (other / "y.manifest").read_text()


def test_manifest_grammar_edges(tmp_path):
    from paper_2303_09523_b200.errors import ManifestParse
    from paper_2303_09523_b200.stack_io import parse_manifest
    p = tmp_path / "m.manifest"
    p.write_text("# header\n\n  pixel_spacing_mm = 0.5   0.7 # trailing\nslice_gap_mm=3\naxis = coronal\n"
                 "slice = a.png\nslice = sub/b.png\nslice = key = odd.png\n")
    m = parse_manifest(p)
    assert m.pixel_spacing_mm == (0.5, 0.7) and m.slice_gap_mm == 3.0 and m.axis_label == "coronal"
    assert [str(f) for f in m.slice_files] == [str((tmp_path / n).resolve()) for n in
                                                 ("a.png", "sub/b.png", "key = odd.png")]
    with pytest.raises(ManifestParse, match="cannot read manifest"):
        parse_manifest(tmp_path / "absent.manifest")


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted")
def test_manifest_parse_matches_live_reference(tmp_path):
    import subprocess
    import sys
    from paper_2303_09523_b200.stack_io import parse_manifest
    p = tmp_path / "m.manifest"
    p.write_text("pixel_spacing_mm = 1.25 0.75\nslice_gap_mm = 4.5 # c\naxis = sagittal\n"
                 "slice = x/../a.png\nslice = b.png\n")
    code = ("import sys, json; from volkrig.io import parse_manifest as P; m = P(sys.argv[1]);"
            "print(json.dumps([list(map(str, m.slice_files)), list(m.pixel_spacing_mm), m.slice_gap_mm, m.axis_label]))")
    out = subprocess.run([sys.executable, "-c", code, str(p)], env={**os.environ, "PYTHONPATH": REF_SRC},
                         capture_output=True, text=True, check=True).stdout
    ref = json.loads(out)
    m = parse_manifest(p)
    assert [list(map(str, m.slice_files)), list(m.pixel_spacing_mm), m.slice_gap_mm, m.axis_label] == ref
