"""Regenerates tests/golden/*.npz from the reference itself.

TEST INFRASTRUCTURE ONLY. Runs oracle/_ref/ref_dump (built by oracle/Makefile
from the unmodified reference sources) for each fixture configuration below
and stores the resulting arrays as compressed npz files. Usage:
    make -C oracle && python oracle/make_golden.py
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import mtfa  # noqa: E402

REF_DUMP = os.path.join(HERE, "_ref", "ref_dump")
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

TINY_GEN = ["--users", "8", "--scen", "4", "--nh", "2", "--nr", "1", "--lenmin", "0", "--lenmax", "21",
            "--expmin", "0", "--expmax", "2", "--gseed", "1"]
TINY_MODEL = ["--d", "64", "--H", "4", "--G", "2", "--demb", "16", "--E", "4", "--dexp", "64", "--mseed", "7"]

FIXTURES = {
    # verify.hpp:230-289 micro fixtures (micro_schemas/micro_model_config/micro_sample)
    "micro": (["--preset", "micro", "--params", "--dumpx", "1"], True),
    # SURVEY §8(d) tiny: 2 layers = (1:1)x1, d=64, 4Q/2KV, 8 users <=63 context + <=8 targets
    "tiny": (TINY_GEN + TINY_MODEL + ["--blocks", "1", "--K", "1", "--P", "1", "--params", "--dumpx", "8"], True),
    # norm / GQA / stack-shape variants over the same users
    "tiny_seqlen_mqa": (TINY_GEN + TINY_MODEL[:2] + ["--H", "4", "--G", "1", "--demb", "16", "--E", "4",
                        "--dexp", "64", "--mseed", "9", "--blocks", "1", "--K", "3", "--P", "1",
                        "--norm", "seqlen", "--dumpx", "2"], True),
    "tiny_none_mha": (TINY_GEN + ["--d", "64", "--H", "4", "--G", "4", "--demb", "16", "--E", "2", "--dexp", "32",
                      "--mseed", "11", "--blocks", "2", "--K", "0", "--P", "1", "--norm", "none",
                      "--dumpx", "2"], True),
    "tiny_lazy": (TINY_GEN[:-2] + ["--gseed", "5", "--d", "32", "--H", "2", "--G", "1", "--demb", "8", "--E", "3",
                  "--dexp", "16", "--mseed", "13", "--blocks", "1", "--K", "3", "--P", "0",
                  "--dumpx", "2"], True),
    # MTFM-small shape (d=256, 8Q/2KV, (3:1)x1, 448 H + 64 R + 32 T), 4 users; params via init port
    "small4": (["--users", "4", "--scen", "4", "--nh", "2", "--nr", "1", "--lenmin", "224", "--lenmax", "224",
                "--rlen", "64", "--expmin", "8", "--expmax", "8", "--gseed", "3", "--d", "256", "--blocks", "1",
                "--K", "3", "--P", "1", "--H", "8", "--G", "2", "--demb", "16", "--E", "4", "--dexp", "256",
                "--mseed", "7"], False),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, (args, keep_x) in FIXTURES.items():
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, name + ".bin")
            subprocess.run([REF_DUMP, "--out", path] + args, check=True)
            arrs = mtfa.read(path)
        if not keep_x:
            arrs = {k: v for k, v in arrs.items() if not k.startswith("fwd/")}
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **{k.replace("/", "__"): v for k, v in arrs.items()})
        print(name, os.path.getsize(os.path.join(OUT, name + ".npz")))


if __name__ == "__main__":
    main()
