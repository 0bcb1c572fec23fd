"""Seeded synthetic inputs shared by the tests, the bench and the oracle legs.

Holds none of the method's arithmetic: only random matrices shaped like the
paper's workloads.

* ``phi`` family: a_ij = (rand - 0.5) * exp(randn * phi), rand uniform
  in (0, 1] (drawn as 1 - U[0, 1)), randn standard normal; phi controls the spread
  of magnitudes.
* ``uniform`` family (BASELINE.json config 1): uniform in [-1, 1) (2u - 1).
* ``int`` family: integers uniform in [-2^20, 2^20].

Host (numpy) generators use ``numpy.random.Generator(PCG64(seed))``; the device
generator uses ``torch.Generator(device)`` and is used only where the host copy of
the same bits is then handed to the oracle.
"""
import numpy as np


def gen_host(rows: int, cols: int, kind: str = "phi", phi: float = 1.0, seed: int = 0,
             order: str = "F") -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "phi":
        u = 1.0 - rng.random((rows, cols))
        g = rng.standard_normal((rows, cols))
        x = (u - 0.5) * np.exp(g * phi)
    elif kind == "uniform":
        x = 2.0 * rng.random((rows, cols)) - 1.0
    elif kind == "int":
        x = rng.integers(-(2 ** 20), 2 ** 20 + 1, size=(rows, cols)).astype(np.float64)
    elif kind == "normal":
        x = rng.standard_normal((rows, cols))
    else:
        raise ValueError(kind)
    return np.asarray(x, dtype=np.float64, order=order)


def gen_device(rows: int, cols: int, kind: str = "phi", phi: float = 1.0, seed: int = 0,
               device: str = "cuda"):
    """Same distributions generated on the device with a seeded torch generator.
    Returns a column-major (Fortran-ordered) float64 tensor view (shape rows x cols,
    strides (1, rows))."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    shape = (cols, rows)          # allocate transposed, return the transposed view
    if kind == "phi":
        u = 1.0 - torch.rand(shape, generator=g, device=device, dtype=torch.float64)
        n = torch.randn(shape, generator=g, device=device, dtype=torch.float64)
        x = (u - 0.5) * torch.exp(n * phi)
    elif kind == "uniform":
        x = 2.0 * torch.rand(shape, generator=g, device=device, dtype=torch.float64) - 1.0
    elif kind == "normal":
        x = torch.randn(shape, generator=g, device=device, dtype=torch.float64)
    else:
        raise ValueError(kind)
    return x.t()
