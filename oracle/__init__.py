"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this package, and only as the checker.  The product path
(paper_2103_16898_b200) never imports it and fails loudly without its CUDA library.

Contents:
  gcm_ref.c       AES-256-GCM restatement (SP 800-38D) of covault.crypto.aead_open/seal
  logistic_ref.c  fp64 restatement of covault.workload.run_training
  cnn_ref.py      PyTorch-CPU restatement of the paper-shaped CNNs (no reference code
                  exists for them -- parity unpinned against the reference)
"""
