"""Generate slice-stack fixtures and the LIVE reference's load_stack output
(volkrig.io.parse_manifest / _decode_slice / load_stack, io.py:53-143, and
model.normalize_stack, model.py:189-202), run in the build container where
/root/reference is mounted:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_stack.py

Writes small images + manifests under tests/golden/stack/ and the expected
stacks / error classes to tests/golden/reference_stack.npz (+ .json).  Error
messages carry absolute paths; the directory is stored as "{dir}" so the
tests can compare on any machine.  The GPU box never reads /root/reference.
"""

import json
import os
import shutil
import sys

import numpy as np
from PIL import Image

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "stack")


def _phantom(r, n, h, w, hi):
    b = r.normal(size=(n, h, w)).cumsum(1).cumsum(2)
    b = (b - b.min()) / (b.max() - b.min())
    return np.rint(b * hi)


def _write(name, arrs_modes, spacing="0.9 0.9", gap="2.7", axis="axial", ext=".png", extra=""):
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    lines = [f"# fixture {name}", f"pixel_spacing_mm = {spacing}", f"slice_gap_mm = {gap}", f"axis = {axis}"]
    for i, (img, e) in enumerate(arrs_modes):
        fn = f"s{i:03d}{e or ext}"
        img.save(os.path.join(d, fn))
        lines.append(f"slice = {fn}   # slice {i}")
    with open(os.path.join(d, "stack.manifest"), "w") as f:
        f.write("\n".join(lines) + "\n" + extra)
    return os.path.join(d, "stack.manifest")


def fixtures():
    r = np.random.default_rng(108)
    out = []
    a = _phantom(r, 4, 20, 24, 255).astype(np.uint8)
    out.append(("u8_L", [(Image.fromarray(x, "L"), None) for x in a]))
    a = _phantom(r, 3, 17, 23, 4095).astype(np.uint16) + 300
    out.append(("u16_I16", [(Image.fromarray(x), None) for x in a]))
    a = _phantom(r, 3, 16, 18, 70000).astype(np.int32) - 5
    out.append(("i32_I_tiff", [(Image.fromarray(x, "I"), ".tif") for x in a]))
    a = _phantom(r, 5, 12, 15, 255).astype(np.uint8)
    rgb = np.stack([a[3], 255 - a[3], a[3] // 2], -1).astype(np.uint8)
    mixed = [(Image.fromarray(a[0], "L"), None),
             (Image.fromarray(a[1], "L").convert("P"), None),
             (Image.fromarray(a[2] > 128), None),
             (Image.fromarray(rgb, "RGB"), None),
             (Image.fromarray((a[4].astype(np.uint16) * 257)), None)]
    out.append(("mixed_modes", mixed))
    c = np.full((12, 10), 77, np.uint8)
    out.append(("constant", [(Image.fromarray(c, "L"), None) for _ in range(3)]))
    return out


def error_cases():
    """(name, manifest text or None, files {name: PIL image or bytes})."""
    r = np.random.default_rng(143)
    img = lambda h, w: Image.fromarray(r.integers(0, 255, (h, w)).astype(np.uint8), "L")
    base = "pixel_spacing_mm = 1.0 1.0\nslice_gap_mm = 5.0\n"
    return [
        ("no_equals", base + "slice s0.png\n", {"s0.png": img(4, 5)}),
        ("one_spacing", "pixel_spacing_mm = 1.0\nslice_gap_mm = 5.0\nslice = s0.png\n", {"s0.png": img(4, 5)}),
        ("bad_axis", base + "axis = oblique\nslice = s0.png\n", {"s0.png": img(4, 5)}),
        ("unknown_key", base + "thickness = 2\n", {}),
        ("no_gap", "pixel_spacing_mm = 1.0 1.0\nslice = s0.png\nslice = s1.png\n", {}),
        ("no_slices", base, {}),
        ("duplicate", base + "slice = s0.png\nslice = ./s0.png\n", {"s0.png": img(4, 5)}),
        ("dims", base + "slice = s0.png\nslice = s1.png\nslice = s2.png\n",
         {"s0.png": img(4, 5), "s1.png": img(4, 5), "s2.png": img(5, 4)}),
        ("dims_before_decode", base + "slice = s0.png\nslice = s1.png\nslice = s2.png\n",
         {"s0.png": img(4, 5), "s1.png": img(6, 5), "s2.png": b"not an image"}),
        ("not_image", base + "slice = s0.png\nslice = s1.png\n", {"s0.png": img(4, 5), "s1.png": b"\x89PNG junk"}),
        ("missing_file", base + "slice = s0.png\nslice = gone.png\n", {"s0.png": img(4, 5)}),
        ("single_slice", base + "slice = s0.png\n", {"s0.png": img(4, 5)}),
        ("bad_float", "pixel_spacing_mm = 1.0 x\nslice_gap_mm = 5.0\nslice = s0.png\n", {"s0.png": img(4, 5)}),
        ("zero_gap", "pixel_spacing_mm = 1.0 1.0\nslice_gap_mm = 0\nslice = s0.png\nslice = s1.png\n",
         {"s0.png": img(4, 5), "s1.png": img(4, 5)}),
    ]


def main():
    from volkrig import io as RIO
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    blob, meta = {}, {"stacks": [], "errors": []}
    for name, imgs in fixtures():
        man = _write(name, imgs)
        st = RIO.load_stack(man)
        modes = []
        for f in RIO.parse_manifest(man).slice_files:
            with Image.open(f) as im:
                modes.append(im.mode)
        blob[f"{name}/slices"] = st.slices
        meta["stacks"].append({"name": name, "manifest": os.path.relpath(man, HERE), "modes": modes,
                               "pixel_spacing": list(st.pixel_spacing), "slice_gap_mm": st.slice_gap_mm,
                               "axis_label": st.axis_label, "shape": list(st.slices.shape)})
    for name, text, files in error_cases():
        d = os.path.join(OUT, "err_" + name)
        os.makedirs(d)
        for fn, content in files.items():
            if isinstance(content, bytes):
                with open(os.path.join(d, fn), "wb") as f:
                    f.write(content)
            else:
                content.save(os.path.join(d, fn))
        man = os.path.join(d, "stack.manifest")
        with open(man, "w") as f:
            f.write(text)
        try:
            RIO.load_stack(man)
            cls, msg = None, None
        except Exception as e:      # noqa: BLE001 -- recording the reference's contract
            cls, msg = type(e).__name__, str(e).replace(os.path.realpath(d), "{dir}")
        meta["errors"].append({"name": name, "manifest": os.path.relpath(man, HERE), "error": cls,
                               "message": msg})
    # write_manifest round trip (io.py:93-105)
    m = RIO.parse_manifest(os.path.join(OUT, "u8_L", "stack.manifest"))
    wpath = os.path.join(OUT, "u8_L", "rewritten.manifest")
    RIO.write_manifest(m, wpath)
    with open(wpath) as f:
        meta["write_manifest"] = {"source": "stack/u8_L/stack.manifest", "text": f.read()}
    os.remove(wpath)
    import PIL
    meta["env"] = {"numpy": np.__version__, "pillow": PIL.__version__, "python": sys.version.split()[0]}
    np.savez_compressed(os.path.join(HERE, "reference_stack.npz"), **blob)
    with open(os.path.join(HERE, "reference_stack.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
