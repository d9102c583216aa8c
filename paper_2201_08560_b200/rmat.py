"""Synthetic Graph500-style R-MAT graphs generated on the device.

The reference ships no generator; this one fixes the input
for every benchmark: Kronecker/R-MAT with (a, b, c, d) = (.57, .19, .19, .05),
``edgefactor * 2**scale`` edges, a keyed bijective vertex permutation, then
(for undirected graphs) symmetrised, self-loops dropped and de-duplicated
with CsrMatrix.from_coo semantics -- all on the GPU (csrc/rmat.cu: counter
based splitmix64 stream, radix sort, unique).  oracle.rmat_csr is the CPU
twin that produces the identical graph.
"""

from __future__ import annotations

from . import _capi
from . import _device as dev
from .formats import CsrMatrix, coo_to_csr_device


def rmat_edges(scale: int, edgefactor: int = 16, seed: int = 1):
    """(src, dst) int32 CUDA tensors of ``edgefactor << scale`` generated edges."""
    t = dev.require_cuda()
    m = int(edgefactor) << int(scale)
    src = t.empty(m, dtype=t.int32, device=dev.device())
    dst = t.empty(m, dtype=t.int32, device=dev.device())
    _capi.call("b2sr_rmat_edges", int(scale), m, int(seed), src.data_ptr(), dst.data_ptr(), dev.stream())
    return src, dst


def rmat_csr(scale: int, edgefactor: int = 16, seed: int = 1, undirected: bool = True) -> CsrMatrix:
    """Device-resident CSR of an R-MAT graph (host arrays materialise lazily)."""
    src, dst = rmat_edges(scale, edgefactor, seed)
    n = 1 << int(scale)
    csr = coo_to_csr_device(n, src, dst, symmetrize=undirected, drop_loops=undirected)
    del src, dst
    return csr
