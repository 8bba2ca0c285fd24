"""The reference package's own CLI (`twedband twed|batch|...`, pkg/src/twedband/cli.py:23-307)
on the B200 kernels.

    python -m paper_2007_16135_b200.refcli twed a.csv b.csv [--nu ... --lambda ... --json]
    python -m paper_2007_16135_b200.refcli batch DIR [--symmetric] [--out matrix.csv]

It imports the user's installed `twedband`, points its band solvers at libtwb200 through the
S2 seam (`seam.install`, _kernels.py:128,146), and hands `argv` to `twedband.cli.main`.
Argument parsing, CSV IO (io.py:32-107), exit codes and JSON reports stay the reference's.
Only the DP sweep runs on the GPU.
"""

from __future__ import annotations

import sys


def main(argv=None) -> int:
    try:
        import twedband
        from twedband import cli
    except ImportError as exc:  # the reference package is the user's install
        print(f"refcli: the reference package `twedband` is not importable ({exc})",
              file=sys.stderr)
        return 2
    from . import seam

    seam.install(twedband)
    return int(cli.main(sys.argv[1:] if argv is None else argv) or 0)


if __name__ == "__main__":
    sys.exit(main())
