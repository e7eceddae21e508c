"""Regenerate tests/golden/reference_vectors.npz from the reference itself.

Runs only in the build container (needs /root/reference): compiles gen_golden.cpp against the
reference's headers, its test-support generators and its unmodified Eigen-free sources, runs
it, and packs the raw outputs into one compressed .npz that is committed.

    python tests/golden/make_golden.py
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/proj"
DT = {"u1": np.uint8, "u4": np.uint32, "u8": np.uint64, "i4": np.int32}


def main() -> int:
    if not os.path.isdir(REF):
        print("make_golden: /root/reference is not present", file=sys.stderr)
        return 1
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "gen_golden")
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", f"{REF}/include", "-I", f"{REF}/tests",
                        os.path.join(HERE, "gen_golden.cpp"), f"{REF}/src/zcurve.cpp", f"{REF}/src/pool.cpp",
                        f"{REF}/src/layouts.cpp", f"{REF}/src/image.cpp", "-lpthread", "-o", exe], check=True)
        out = os.path.join(tmp, "out")
        os.makedirs(out)
        subprocess.run([exe, out], check=True)
        arrays = {}
        with open(os.path.join(out, "manifest.txt")) as f:
            for line in f:
                parts = line.split()
                name, dt, shape = parts[0], parts[1], tuple(int(x) for x in parts[2:])
                arrays[name] = np.fromfile(os.path.join(out, name + ".bin"), dtype=DT[dt]).reshape(shape)
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **arrays)
    print(f"wrote {len(arrays)} arrays")
    return 0


if __name__ == "__main__":
    sys.exit(main())
