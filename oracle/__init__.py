"""FP64 CPU oracle for the Morphling GCN training hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import or call
anything in this package.  The product path (`paper_2512_01678_b200`) never
imports it, and this package never imports the product: the two share no code,
no headers, no constant tables.  Inputs come from `synth/` (a generator with
none of the method's arithmetic).

What it computes is the plain mathematical definition of one GCN training
epoch as the paper states the problem (§Background P:89-99,
Alg. 1, Alg. 3, §Distributed Runtime P:508-536), with the
readings of SURVEY.md §8(c) c.3 (Q1-Q28) wherever the paper is silent.

Parity status of each function (pins live in tests/test_oracle_*.py):
  graph_build ........ pinned (hand cases, brute force, invariants, closed forms)
  dinv / a_hat ....... pinned (closed forms K_n, star, regular; row invariants)
  analyze_features ... pinned (paper value s=99.21% NELL P:690, boundary S:147-149)
  xavier_init ........ pinned (splitmix64 known answer, bound, variance)
  philox4x32_10 ...... pinned (Random123 known-answer vectors)
  aggregate .......... pinned (brute-force dense Â, identity, Â·sqrt(d)=sqrt(d))
  forward/backward ... pinned (central finite differences, torch.float64 autograd)
  softmax_ce ......... pinned (uniform logits -> ln C, C=2 logistic, torch CE)
  adam_step .......... pinned (first step -lr*sign(g), zero grad, torch.optim.Adam)
  train .............. pinned (monotone loss on the separable SBM toy)
  partition_1d / localize ... pinned (brute-force recount, union = global set)
  tf32_rna ........... pinned (known values incl. ties away from zero, bounds, idempotence)
  bf16_rne ........... pinned (known values incl. ties to even, bounds, idempotence, torch bf16)
  aggregate_scheme (sum/mean) ... pinned (brute force over neighbour sets from the raw edge list,
                                  dense adjoints, Ã·1 = d̃, mean of a constant, torch autograd)
  aggregate_max / _backward ..... pinned (brute force with ties -> smallest id, hand star case,
                                  central differences, routed-mass conservation)
  forward/backward (sum/mean/max) pinned (central finite differences of the whole loss)
  sgd_step / adamw_step ......... pinned (closed forms; torch.optim.SGD / AdamW traces)
  partition_greedy / _components / relabel / partition_stats ... pinned (hand-worked star and
                                  component cases, scipy connected components, the greedy's
                                  list-scheduling bound, brute-force recounts, permutation
                                  invariance of training under relabelling)
  bounds.tf32_gradient_bounds ... a test tolerance, not an oracle result; pinned by an FP32
                                  emulation of the GPU's arithmetic staying inside it while the
                                  bound stays tight (tests/test_oracle_bounds.py)
  absolute model quality vs the paper ... parity unpinned (the paper prints no loss
                                           or accuracy value)
"""
from .gcn_oracle import *  # noqa: F401,F403
from .bounds import FLOOR_REL, tf32_gradient_bounds  # noqa: F401
