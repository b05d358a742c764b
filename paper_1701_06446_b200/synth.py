"""Seeded synthetic row streams for the five BASELINE.json configurations.

BASELINE.json names no public dataset and the reference's own generator
(copula_gen.cpp) does not produce these distributions, so the streams are
defined here.  Rows arrive in order: the first window is rows
[0, T), step k (1-based) brings rows [T + (k-1) p, T + k p).

Readings of the config text that needed a choice:
  * cfg1: the Student-t(nu=5) block uses Sigma[0:16,0:16] as the SCALE matrix
    (covariance = nu/(nu-2) * Sigma): z ~ N(0, Sigma_16), w ~ chi2(5),
    t = z / sqrt(w / 5).  Steps 1-25 are Gaussian, 26-50 t on columns 0-15.
  * cfg2: each entry is independently replaced, with probability 0.1, by a
    Laplace(0, 1) draw.
  * cfg3: Gaussian with a seeded random correlation matrix built as A A^T
    with A ~ U(-1,1)^{n x n}, normalised to unit diagonal.
  * cfg4: from step 5 on, columns 0-47 switch to t(nu=4) with the same
    Gaussian scale.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED = 1701064460


@dataclass(frozen=True)
class Config:
    index: int
    d: int
    n: int
    b: int
    T: int
    p: int
    steps: int
    name: str

    @property
    def rows_total(self) -> int:
        return self.T + self.p * self.steps


CONFIGS = [
    Config(0, 4, 24, 3, 5000, 500, 20, "cfg0_d4_n24_b3_T5000_p500"),
    Config(1, 4, 96, 8, 20000, 1000, 50, "cfg1_d4_n96_b8_T20000_p1000"),
    Config(2, 6, 48, 4, 50000, 2000, 20, "cfg2_d6_n48_b4_T50000_p2000"),
    Config(3, 4, 256, 16, 100000, 4096, 20, "cfg3_d4_n256_b16_T100000_p4096"),
    Config(4, 6, 96, 8, 200000, 8192, 10, "cfg4_d6_n96_b8_T200000_p8192"),
]


def _sigma_llt(rng: np.random.Generator, n: int) -> np.ndarray:
    L = rng.uniform(-1.0, 1.0, (n, n))
    return L @ L.T + 0.5 * np.eye(n)


def _corr_aat(rng: np.random.Generator, n: int) -> np.ndarray:
    A = rng.uniform(-1.0, 1.0, (n, n))
    S = A @ A.T
    d = np.sqrt(np.diag(S))
    return S / np.outer(d, d)


class StreamGen:
    """Generates the row stream of one config lazily, batch by batch."""

    def __init__(self, cfg: Config, seed: int = SEED):
        self.cfg = cfg
        self.rng = np.random.default_rng([seed, cfg.index])
        n = cfg.n
        if cfg.index == 3:
            self.sigma = _corr_aat(self.rng, n)
        else:
            self.sigma = _sigma_llt(self.rng, n)
        self.chol = np.linalg.cholesky(self.sigma)

    def _gauss(self, rows: int) -> np.ndarray:
        return self.rng.standard_normal((rows, self.cfg.n)) @ self.chol.T

    def _t_block(self, z: np.ndarray, cols: slice, nu: float) -> None:
        w = self.rng.chisquare(nu, (z.shape[0], 1))
        z[:, cols] = z[:, cols] / np.sqrt(w / nu)

    def window(self) -> np.ndarray:
        """The first T rows."""
        return self._rows(self.cfg.T, step=0)

    def batch(self, step: int) -> np.ndarray:
        """The p incoming rows of step `step` (1-based)."""
        return self._rows(self.cfg.p, step=step)

    def _rows(self, rows: int, step: int) -> np.ndarray:
        c = self.cfg
        x = self._gauss(rows)
        if c.index == 1 and step >= 26:
            self._t_block(x, slice(0, 16), 5.0)
        elif c.index == 2:
            m = self.rng.random(x.shape) < 0.1
            x[m] = self.rng.laplace(0.0, 1.0, int(m.sum()))
        elif c.index == 4 and step >= 5:
            self._t_block(x, slice(0, 48), 4.0)
        return np.ascontiguousarray(x)


def stream_rows(cfg: Config, steps: int | None = None, seed: int = SEED) -> np.ndarray:
    """The whole stream (first window + `steps` batches) as one array."""
    g = StreamGen(cfg, seed)
    steps = cfg.steps if steps is None else steps
    return np.concatenate([g.window()] + [g.batch(k) for k in range(1, steps + 1)])
