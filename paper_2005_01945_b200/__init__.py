"""B200-native TFHE gate-evaluation engine behind the `encirc` GateEngine API.

Drop-in for the evaluation path of the reference package (arXiv 2005.01945's
`encirc`): key generation, encrypt/decrypt, bootstrapped boolean gates and the
add / multiply / vector / matrix circuits keep the reference's names and
semantics; `B200Engine` replaces `OracleBootstrapEngine` with real TFHE gate
bootstrapping on the GPU (hand-written sm_100a kernels behind the C ABI in
include/tfhe_b200.h).  Importing this package does not need a GPU;
constructing a `B200Engine` does, and there is no CPU fallback.
"""

from .datasets import (
    KIND_BINARY,
    KIND_NUMERICAL,
    KINDS,
    Dataset,
    DatasetFormatError,
    read_csv,
    synthesize,
    to_csv_text,
    write_csv,
)
from .engine import (
    TWO_INPUT_KINDS,
    B200Engine,
    BootstrapMarginError,
    EncBit,
    GateEngine,
    GateKind,
    GateStats,
    ReferenceEngine,
    truth_table,
)
from .integers import (
    KARATSUBA_MIN_WIDTH,
    EncryptedInt,
    accumulate_tree,
    add_bitwise,
    add_numberwise,
    as_signed,
    complement,
    decrypt_int,
    encrypt_int,
    mul_karatsuba,
    mul_naive,
    negate,
    shift_left,
    trivial_int,
    truncate,
    zero_extend,
)
from .keys import EvaluationKeys, RingParams, generate_evaluation_keys
from .linalg import (
    DEFAULT_FLAT_JOB_CEILING,
    EncryptedIntVector,
    EncryptedMatrix,
    FlatLaunchTooLarge,
    decrypt_matrix,
    decrypt_vector,
    encrypt_matrix,
    encrypt_vector,
    mat_add,
    mat_mul_cannon,
    mat_mul_flat,
    vec_add,
    vec_mul,
)
from .serialize import (
    FormatError,
    dump_eval_keys,
    dump_int,
    dump_key,
    dump_matrix,
    dump_params,
    dump_sample,
    dump_vector,
    load_eval_keys,
    load_int,
    load_key,
    load_key_file,
    load_matrix,
    load_params,
    load_sample,
    load_vector,
    save_key,
)
from .regression import (
    DEFAULT_BITS,
    RegressionReport,
    SingularSystemError,
    VerificationError,
    fit_encrypted,
    solve_exact,
)
from .scheduler import DEFAULT_MAX_BATCH, PARALLEL_BLOCK, JobBatch, PoolConfig, WorkerPool
from .torus import (
    DEFAULT_ALPHA,
    DEFAULT_M,
    DEFAULT_W,
    DecryptionUnreliableError,
    LweParams,
    LweSample,
    SecretKey,
    TorusElement,
    decrypt_bit,
    encrypt_bit,
    keygen,
    lwe_linear,
    phase,
    trivial_sample,
)

__version__ = "0.1.0"
