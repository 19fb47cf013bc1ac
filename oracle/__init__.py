"""CPU oracle for the SAGA-NN layer hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/sagastream/tensor.py` primitives composed per the
SPEC's SAGA-NN layer, partitioner and stage-op contracts).  It is the checker,
never the product:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_1810_08403_b200`` never imports it and fails
  loudly when its CUDA library is missing.

Parity is pinned: ``tests/golden/make_golden.py`` runs the *real* reference
``tensor.py`` (Tensor/Tape) on small GCN / G-GCN graphs and commits the
outputs as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
oracle against them bit for bit, and ``tests/test_oracle_kat.py`` restates the
reference unit tests (``pkg/tests/test_tensor.py``) and the SPEC known-answer
examples against it.

Modules
-------
primitives  tensor.py ops as pure numpy functions (fwd + explicit bwd).
rng         counter-based splitmix64 generator shared bit-for-bit with the C++/CUDA
            generators (synthetic graphs and features).
graph       degrees, GCN edge weights, reencode_balance, partition_2d, split plan.
saga        GCN / G-GCN layers: dense (reference composition) and chunked
            (Locality order, subgroup-split gather) forward + backward, 2-layer epoch.
"""
