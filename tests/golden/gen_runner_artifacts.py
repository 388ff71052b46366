"""Generate runner artifacts (manifest + TWT1 tensors) with the REFERENCE CLI
(`tiledsl emit` + `tiledsl simulate --save-dir`, cli.py:194-231, 274-291), as
its own runner tests do (triton_runner/tests/test_runner.py:40-57).  Build
container only; the outputs are committed under tests/golden/runner/."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "runner"
CASES = {
    "add": {"N": 10, "BLOCK_SIZE": 4},
    "mm": {"M": 4, "N": 6, "K": 5, "BLOCK_SIZE_M": 2, "BLOCK_SIZE_N": 2, "BLOCK_SIZE_K": 2},
    "addmm": {"M": 8, "N": 8, "K": 16, "BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 8},
    "softmax": {"R": 6, "C": 20, "COLS_PADDED": 32},
    "conv2d": {"N": 1, "C": 2, "H": 5, "W": 6, "K": 3, "R": 3, "S": 2,
               "BLOCK_SIZE_M": 4, "BLOCK_SIZE_N": 4, "BLOCK_SIZE_K": 4},
}


def main():
    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src", PYTHONHASHSEED="0")
    shutil.rmtree(OUT, ignore_errors=True)
    for kernel, binds in CASES.items():
        d = OUT / kernel
        d.mkdir(parents=True)
        run = lambda *a: subprocess.run([sys.executable, "-m", "tiledsl", *a], env=env, check=True,
                                        capture_output=True, text=True)
        run("emit", kernel, "-o", str(d / f"{kernel}.py"))
        (d / f"{kernel}.py").unlink()        # Triton source not needed by the B200 runner
        run("simulate", kernel, "--bind", ",".join(f"{k}={v}" for k, v in binds.items()),
            "--save-dir", str(d))
    print("written", sorted(p.relative_to(OUT).as_posix() for p in OUT.rglob("*")))


if __name__ == "__main__":
    main()
