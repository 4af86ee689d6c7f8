"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs oracle/_ref/impm_ref (the unmodified reference core built by
oracle/Makefile from /root/reference/proj/src) on every spec in
tests/golden/specs/ and packs the per-stage arrays it writes into
tests/golden/<spec>.npz. Also packs the reference's own committed outputs
(/root/reference/proj/out/*/*.csv) into tests/golden/reference_out.npz.

Only runs in the build container (needs /root/reference); the fixtures it
writes are committed so the GPU box never reads /root/reference.

    python tests/golden/make_golden.py [spec ...]
"""
import glob
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_TOOL = os.path.join(REPO, "oracle", "_ref", "impm_ref")
REF_OUT = "/root/reference/proj/out"

# big per-case arrays that are not needed for fixtures above this many rows
SKIP_IF_LARGE = {"J1_vals": 200_000, "delta1": 200_000, "particles_step1": 200_000, "particles_commit1": 200_000}


def make_case(spec_path):
    name = os.path.splitext(os.path.basename(spec_path))[0]
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([REF_TOOL, "dump", spec_path, tmp], check=True)
        arrays = {}
        for f in sorted(glob.glob(os.path.join(tmp, "*.npy"))):
            key = os.path.splitext(os.path.basename(f))[0]
            a = np.load(f)
            if key in SKIP_IF_LARGE and a.size > SKIP_IF_LARGE[key]:
                continue
            arrays[key] = a
        with open(spec_path) as fh:
            arrays["spec"] = np.frombuffer(fh.read().encode(), dtype=np.uint8)
    out = os.path.join(HERE, name + ".npz")
    np.savez_compressed(out, **arrays)
    print(f"{name}: {len(arrays)} arrays, {os.path.getsize(out) / 1024:.0f} KiB")


def pack_reference_out():
    arrays = {}
    for csv in sorted(glob.glob(os.path.join(REF_OUT, "*", "*.csv"))):
        scen = os.path.basename(os.path.dirname(csv))
        key = scen + "__" + os.path.splitext(os.path.basename(csv))[0]
        with open(csv) as fh:
            header = fh.readline().strip()
        try:
            data = np.loadtxt(csv, delimiter=",", skiprows=1, ndmin=2)
        except ValueError:
            continue  # non-numeric columns (jacobian_bench strategy names)
        arrays[key] = data
        arrays[key + "__header"] = np.frombuffer(header.encode(), dtype=np.uint8)
    out = os.path.join(HERE, "reference_out.npz")
    np.savez_compressed(out, **arrays)
    print(f"reference_out: {len(arrays) // 2} csvs, {os.path.getsize(out) / 1024:.0f} KiB")


def main():
    if not os.path.exists(REF_TOOL):
        subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "ref"], check=True)
    specs = sys.argv[1:] or sorted(glob.glob(os.path.join(HERE, "specs", "*.spec")))
    for s in specs:
        make_case(s if os.path.exists(s) else os.path.join(HERE, "specs", s + ".spec"))
    if not sys.argv[1:]:
        pack_reference_out()


if __name__ == "__main__":
    main()
