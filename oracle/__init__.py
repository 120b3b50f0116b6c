"""CPU oracle for the ShiftAddViT inference hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the forward semantics of the reference
package `shiftadd` (arXiv 2306.06446 desk artefact, /root/reference/pkg/src):
sign binarization, shift quantization, the binary Q(KV) attention core, the
token-grid depthwise conv, the top-1 two-expert router / dispatch, and the
layer/model forward passes, plus the PVT / DeiT compositions built from those
layers.

Every function cites the reference file:line it follows. Parity of this
restatement is PINNED against golden vectors produced by importing the real
reference in the build container (tests/golden/make_golden.py →
tests/golden/*.npz; checked by tests/test_oracle_golden.py).

Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` may import this package, and only as the checker
or the timed CPU reference. The product (`paper_2306_06446_b200`) never
imports it.
"""

from . import ops, nets  # noqa: F401
