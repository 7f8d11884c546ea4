"""Binary volume format, host-side checks (io.py:170-186) on golden files the
live reference wrote (tests/golden/make_golden_volio.py) -- CPU only."""

import os
import struct

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _blob(k="a"):
    with open(os.path.join(HERE, "golden", f"ref_volume_{k}.vkv"), "rb") as f:
        return f.read()


def test_header_of_reference_files():
    from paper_2303_09523_b200.volume_io import parse_header
    assert parse_header(_blob("a")) == ((7, 6, 5), (1, -2, 3))
    assert parse_header(_blob("b")) == ((7, 5, 3), (0, 0, 0))
    assert parse_header(_blob("c")) == ((3, 4, 9), (-7, 11, 2 ** 20))


@pytest.mark.parametrize("mutate,match", [
    (lambda b: b[:20], "truncated"),
    (lambda b: b"VOLKRIX\x00" + b[8:], "bad magic"),
    (lambda b: b[:8] + struct.pack("<I", 2) + b[12:], "unsupported volume version 2"),
    (lambda b: b[:-1], "size"),
    (lambda b: b + b"\x00", "size"),
])
def test_corrupt_headers(mutate, match):
    from paper_2303_09523_b200.errors import CorruptHeader
    from paper_2303_09523_b200.volume_io import parse_header
    with pytest.raises(CorruptHeader, match=match):
        parse_header(mutate(_blob("a")))


def test_missing_file_is_io_error(tmp_path):
    from paper_2303_09523_b200.errors import Io
    from paper_2303_09523_b200.volume_io import load_volume
    with pytest.raises(Io):
        load_volume(tmp_path / "nope.vkv")
