"""Stream configurations C1-C5 (BASELINE.json ``configs``) plus small test variants.

Each record states the shape, ranks, batching and noise of one synthetic stream, as
read in SURVEY.md §8(d).1 and DESIGN.md "Input recipe".  Dimensions use the paper's
notation: modes 1..N-1 are the non-temporal modes with sizes I_1..I_{N-1}; mode N is
time.  ``ranks`` = (R_1, ..., R_N) with R_{N+1} = R_1.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Tuple


@dataclass(frozen=True)
class StreamConfig:
    name: str
    dims: Tuple[int, ...]            # I_1 .. I_{N-1}
    ranks: Tuple[int, ...]           # R_1 .. R_N
    t_init: int                      # temporal length of X_init
    t_new: int                       # temporal length of every X_new
    n_batches: int                   # number of update steps
    dtype: str                       # 'f64' or 'f32' storage of X
    contract: str                    # 'f64' or '3xtf32' contraction precision on the GPU
    kind: str = "tr"                 # 'tr' (exact TR + noise) or 'video' (C3 blobs)
    core_scale: float = 1.0          # std of true-core entries
    noise_abs: float = 0.0           # absolute noise std (applied to every entry)
    variant: str = "det"             # 'det', 'uniform', 'leverage'
    sketch_rows: int = 0             # m for rSTR
    seed: int = 0
    init_perturb: float = 1e-2       # relative perturbation of truth-based init cores
    split_k: int = 0                 # two-pass split point k (0 = automatic)
    notes: str = ""

    @property
    def N(self) -> int:
        return len(self.dims) + 1

    @property
    def T_total(self) -> int:
        return self.t_init + self.t_new * self.n_batches

    @property
    def slice_entries(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n

    @property
    def batch_entries(self) -> int:
        return self.slice_entries * self.t_new

    def with_(self, **kw) -> "StreamConfig":
        return replace(self, **kw)


def _rms_tr(R: int, sigma_c: float, N: int) -> float:
    # RMS of an entry of TR(G_1..G_N) with i.i.d. N(0, sigma_c^2) cores of uniform rank R:
    # E[X^2] = (R sigma_c^2)^N.
    return (R * sigma_c ** 2) ** (N / 2.0)


CONFIGS = {
    # configs[0]: order-3 20x20xT fp64, ranks (3,3,3), N(0,1) cores, 1e-3 absolute noise.
    "C1": StreamConfig("C1", (20, 20), (3, 3, 3), 10, 2, 10, "f64", "f64",
                       core_scale=1.0, noise_abs=1e-3, seed=101),
    # configs[1]: order-4 60^3xT fp32, R=5, cores N(0,1)/sqrt(5), SNR 40 dB -> sigma = 0.01*RMS.
    "C2": StreamConfig("C2", (60, 60, 60), (5, 5, 5, 5), 20, 5, 36, "f32", "3xtf32",
                       core_scale=5 ** -0.5, noise_abs=0.01 * _rms_tr(5, 5 ** -0.5, 4), seed=202),
    # configs[2]: video-shaped 240x320xT fp32, 10 separable sinusoid-modulated blobs in [0,1],
    # 0.01 noise, ranks 10; FP64 contraction.
    "C3": StreamConfig("C3", (240, 320), (10, 10, 10), 50, 10, 95, "f32", "f64",
                       kind="video", noise_abs=0.01, seed=303, init_perturb=5e-2),
    # configs[3]: order-4 100^3xT fp32, R=8, N(0,1) cores, 1e-2 relative noise; rSTR m=2000.
    "C4": StreamConfig("C4", (100, 100, 100), (8, 8, 8, 8), 10, 10, 19, "f32", "3xtf32",
                       core_scale=1.0, noise_abs=1e-2 * _rms_tr(8, 1.0, 4), seed=404,
                       sketch_rows=2000),
    # configs[4]: order-5 40^4xT fp32, R=10, N(0,1) cores, 1e-3 relative noise; sharded on mode 1.
    "C5": StreamConfig("C5", (40, 40, 40, 40), (10, 10, 10, 10, 10), 8, 8, 15, "f32", "3xtf32",
                       core_scale=1.0, noise_abs=1e-3 * _rms_tr(10, 1.0, 5), seed=505, split_k=2),
}

# Small variants for the oracle suite and for GPU parity at sizes the oracle finishes in
# seconds.  Unequal ranks catch index-pairing mistakes; ragged dims span several tiles.
CONFIGS.update({
    "T3": StreamConfig("T3", (6, 4), (2, 3, 4), 6, 2, 3, "f64", "f64",
                       core_scale=1.0, noise_abs=1e-2, seed=7),
    "T4": StreamConfig("T4", (6, 4, 3), (2, 3, 4, 2), 6, 3, 3, "f64", "f64",
                       core_scale=1.0, noise_abs=1e-2, seed=8),
    "T5": StreamConfig("T5", (4, 3, 5, 3), (2, 3, 2, 4, 3), 5, 2, 3, "f64", "f64",
                       core_scale=1.0, noise_abs=1e-2, seed=9, split_k=2),
    # GPU parity sizes: several 128-row tiles plus a ragged tail in every contraction.
    "P2": StreamConfig("P2", (24, 19, 17), (3, 4, 5, 2), 6, 5, 4, "f32", "3xtf32",
                       core_scale=0.5, noise_abs=1e-2, seed=21),
    "P3": StreamConfig("P3", (37, 53), (4, 6, 5), 12, 7, 4, "f32", "f64",
                       kind="tr", core_scale=0.5, noise_abs=1e-2, seed=31),
    "P5": StreamConfig("P5", (12, 11, 9, 7), (3, 4, 5, 3, 4), 5, 3, 3, "f32", "3xtf32",
                       core_scale=0.5, noise_abs=1e-2, seed=51, split_k=2),
    "P1": StreamConfig("P1", (20, 20), (3, 3, 3), 10, 2, 10, "f64", "f64",
                       core_scale=1.0, noise_abs=1e-3, seed=111),
    # Large ranks (R_nR_{n+1} up to 120 = 15 pivot blocks of the inverse, rank 12 > 10 in the
    # table / absorb kernels), ragged dims.
    "P6": StreamConfig("P6", (36, 29, 23), (12, 10, 11, 9), 10, 4, 3, "f32", "3xtf32",
                       core_scale=12 ** -0.5, noise_abs=1e-2, seed=61),
    # rSTR parity: I_k > R_kR_{k+1} so leverage scores are non-uniform; m >= max R_nR_{n+1}.
    # Fused pass-2 table generation (uniform rank R in {4, 8, 10}, k = 2, I_1 >= 32): K-tiles that
    # cross a multiple of I_1 (G4, G10) or align with it (G8), ragged last K-tile and M-tile.
    "G4": StreamConfig("G4", (36, 7, 30, 9), (4, 4, 4, 4, 4), 6, 3, 3, "f32", "3xtf32",
                       core_scale=0.5, noise_abs=1e-2, seed=71, split_k=2),
    "G8": StreamConfig("G8", (32, 5, 20, 8), (8, 8, 8, 8, 8), 6, 3, 3, "f32", "3xtf32",
                       core_scale=8 ** -0.5, noise_abs=1e-2, seed=72, split_k=2),
    "G10": StreamConfig("G10", (40, 6, 13, 11), (10, 10, 10, 10, 10), 6, 2, 3, "f32", "3xtf32",
                        core_scale=10 ** -0.5, noise_abs=1e-2, seed=73, split_k=2),
    "R4": StreamConfig("R4", (30, 25, 20), (2, 3, 2, 3), 6, 4, 3, "f32", "f64",
                       core_scale=0.7, noise_abs=1e-2, seed=41, sketch_rows=200),
    "R5": StreamConfig("R5", (12, 9, 10, 8), (2, 3, 2, 2, 3), 5, 3, 3, "f64", "f64",
                       core_scale=0.7, noise_abs=1e-2, seed=42, sketch_rows=150),
})


def get_config(name: str) -> StreamConfig:
    try:
        return CONFIGS[name]
    except KeyError:
        raise KeyError(f"unknown stream config {name!r}; known: {sorted(CONFIGS)}") from None
