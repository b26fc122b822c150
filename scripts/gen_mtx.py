"""Write a synthetic banded Matrix Market file (bench / smoke input for
`bench.py --workload mtx`; no SuiteSparse download is possible offline)."""
import sys

import numpy as np


def main(path: str, n: int = 300000, k: int = 8, band: int = 2000, seed: int = 5) -> None:
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), k)
    cols = (rows + rng.integers(-band, band, rows.size)) % n
    key = np.unique(rows.astype(np.int64) * n + cols)
    r, c = key // n, key % n
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{n} {n} {r.size}\n")
        np.savetxt(f, np.stack([r + 1, c + 1, rng.uniform(-1, 1, r.size)], 1), fmt="%d %d %.17g")


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:]))
