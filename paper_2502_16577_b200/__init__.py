"""B200-native Gray-walk matrix permanents, drop-in for permkit's hot path.

Same public names and semantics as the reference package permkit
(/root/reference/pkg/src/permkit/__init__.py): ``permanent``, ``perm_nw``,
``perm_spa``, ``permanent_chunked``, ``run_range``, ``execute_plan``,
``reduce_partials`` and the plan / matrix / precision types. The Gray walk
runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/permkit_b200.h; there is no CPU fallback.

    import paper_2502_16577_b200 as permkit
    permkit.permanent([[1, 2], [3, 4]])          # 10 (exact integers)
"""

from .errors import (DecompTimeout, DeviceError, ImpossibleError, ParseError, PermanentError,
                     PolicyError, StructureError)
from .generate import (haar_unitary_block, random_binary, random_real, random_sparse_int,
                       random_sparse_real, random_ternary, uniform)
from .graycode import GrayStep, cbl_sequence, changed_bit, gray_of, subset_columns
from .batch import permanent_batch
from .kernels import perm_nw, perm_spa, total_iterates
from .matrix import (CcsMatrix, CrsMatrix, DenseMatrix, Scalar, SparsePair, coerce_matrix,
                     dense_to_sparse, density, sparse_from_triplets, sparse_to_dense)
from .parallel import (ChunkPlan, HierarchyPlan, PartialResult, cbl_alignment_report,
                       execute_hierarchy, execute_plan, fixed_chunk_plan, init_x_at,
                       initial_product, matrix_content_hash, merge_partial_files,
                       permanent_chunked, plan_chunks, plan_hierarchy, read_partials_file,
                       reduce_partials, run_range, write_partials_file)
from .preprocess import (DecompStats, DmResult, Matching, SingularVerdict, d1compress,
                         d2compress, d34compress, decomp_leaves, decomp_run, decomp_ryser,
                         dm_decompose, dm_filter, max_matching, min_nnz_row_col)
from .precision import (AccumulatorPolicy, DoubleDouble, KahanAccumulator, dd_add, dd_mul,
                        kahan_add, reference_permanent, relative_error, two_prod, two_sum)

__version__ = "0.1.0"


def permanent(matrix, policy="dd", workers: int = 1, aligned: bool = True, *, devices=None):
    """Permanent of rows / numpy array / DenseMatrix / SparsePair (permkit
    __init__.py:109-122). Integer matrices are exact.

    The reference splits the walk over ``workers`` CPU threads; here the walk
    is split into GPU-sized aligned chunks regardless, and ``workers`` > 1
    spreads it over that many GPUs (contiguous Gray-code ranges, fixed-order
    host reduction). ``devices`` selects explicit CUDA ordinals. ``aligned``
    is accepted for compatibility: the GPU split is always the aligned
    (power-of-two) tiling, which permkit's ``aligned=True`` default also uses.
    """
    from . import _native
    from .precision import as_policy
    policy = as_policy(policy)
    m = coerce_matrix(matrix)
    if devices is None and workers > 1:
        devices = list(range(min(workers, _native.device_count())))
    if isinstance(m, SparsePair):
        return perm_spa(m, policy, devices=devices)
    return perm_nw(m, policy, devices=devices)
