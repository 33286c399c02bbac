"""B200-native prover backend for the zkLoRA sumcheck / logUp hot path.

Drop-in entry points (same names, arguments and errors as the reference
package zklora, pkg/src/zklora/*):

  prove_sumcheck(claim, tr)                         sumcheck.py:98
  prove_matmul(a, b, c, key, tr, rng)               gadgets.py:230
  prove_elementprod(a, b, c, key, tr, rng)          gadgets.py:383
  prove_lookup(secret, m, table, key, tr, rng)      lookup.py:143
  compute_multiplicities(entries, table)            lookup.py:91
  batch_inverse(values, p)                          field.py:34
  eq_table(point, p), fold_table(t, r, p)           mle.py:50-82

install() rebinds them inside an importable zklora package so the
reference pipeline and tests run on the GPU unmodified.  All compute runs
in libzkl_b200.so (C-ABI, include/zkl_b200.h); there is no CPU fallback.
"""

from .field import MODULUS, TEST_MODULUS, InversionOfZero, batch_inverse, inverse  # noqa: F401
from .gadgets import (  # noqa: F401
    DeviceMatrix,
    ElementprodProof,
    MatmulProof,
    ProverTensor,
    ShapeMismatch,
    TensorRef,
    matmul_sumcheck,
    matmul_sumcheck_batch,
    prove_elementprod,
    prove_matmul,
    prove_pair_lookup,
)
from .lookup import (  # noqa: F401
    ElementNotInTable,
    LookupProof,
    LookupTable,
    PoleCollision,
    SecretVector,
    compute_multiplicities,
    prove_lookup,
)
from .mle import eq_table, fold_table, mle_evaluate  # noqa: F401
from .nonlinear import (  # noqa: F401
    DigitOutOfRange,
    NormalizationBudgetExceeded,
    PairTable,
    RangeViolation,
    SoftmaxRowProof,
    TableSet,
    prove_rescale,
    prove_rsqrt,
    prove_softmax_row,
    prove_swiglu,
    softmax_row_witness,
)
from .sumcheck import (  # noqa: F401
    DegreeOverflow,
    RoundPolynomial,
    SumcheckClaim,
    SumcheckError,
    SumcheckProof,
    Term,
    prove_sumcheck,
)
from .transcript import Transcript  # noqa: F401


def install(zklora_pkg=None, gpu_commit=False):
    from .install import install as _install

    return _install(zklora_pkg, gpu_commit=gpu_commit)
