"""CPU oracle for the jagged HSTU attention + jagged-CP hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2508_04711_b200`` imports this
package: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (or the timed CPU reference arm), never as the thing measured for the
GPU path.

It is a numpy restatement of the reference package ``jaggedcp``
(``/root/reference/pkg/src/jaggedcp``); every function cites the reference
``file:line`` it follows.  The restatement is *pinned* against the reference
itself: ``tests/golden/make_golden.py`` imports the reference in the build
container and freezes its outputs (attention forward/backward, bucket indices,
plans, permutations, flop counts) into ``tests/golden/*.npz|json``;
``tests/test_oracle_golden.py`` checks this oracle against those fixtures and
against the reference test-suite's known-answer values.
"""

from .attention import (  # noqa: F401
    bucketize_array,
    bucketize,
    compute_bias,
    silu,
    sigmoid,
    hstu_fwd_seq,
    hstu_bwd_seq,
    hstu_forward,
    hstu_backward,
    blockwise_partial,
    normal_init_ts_weights,
)
from .jagged import (  # noqa: F401
    split_even,
    make_minichunks,
    make_contiguous_chunks,
    chunk_assignment,
    chunk_owner_map,
    rank_major_row_order,
    rank_row_ranges,
)
from .cp import build_shard_plan, flops_per_rank, cp_forward_sim  # noqa: F401
from .harness import gen_synthetic_batch, output_errors, concat_batches  # noqa: F401
