"""Regenerate tests/golden/reference_golden.npz from the UNMODIFIED reference.

Runs oracle/_ref/ref_tool (built by `make -C oracle` from /root/reference/proj/src plus
oracle/ref_tool.cpp, which only calls the reference's public API) and packs its raw dumps into
one compressed npz. Run here, in the build container (the GPU box has no /root/reference):

    make -C oracle && python tests/golden/make_golden.py
"""
import json
import pathlib
import subprocess
import sys
import tempfile

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
TOOL = ROOT / "oracle" / "_ref" / "ref_tool"
OUT = pathlib.Path(__file__).resolve().parent / "reference_golden.npz"


def main() -> int:
    if not TOOL.exists():
        print(f"missing {TOOL}; run `make -C oracle` first", file=sys.stderr)
        return 1
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([str(TOOL), "golden", tmp], check=True)
        manifest = json.loads((pathlib.Path(tmp) / "manifest.json").read_text())
        arrays = {}
        for name, meta in manifest.items():
            dtype = {"f64": "<f8", "i64": "<i8"}[meta["dtype"]]
            raw = np.fromfile(pathlib.Path(tmp) / f"{name}.{meta['dtype']}", dtype=dtype)
            arrays[name] = raw.reshape(meta["shape"])
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({len(arrays)} arrays, {OUT.stat().st_size} bytes)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
