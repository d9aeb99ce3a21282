"""CPU oracles for the encrypted-decode hot path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package; the product (paper_2602_11470_b200) never does.

  slot_sim   numpy restatement of the reference SimBackend (engine.cpp)
  layout     restatement of layouts.cpp
  protocols  restatement of vmm.cpp / kv_attention.cpp, generic over a backend
  ckks       ctypes wrapper of ckks_oracle.cpp: the bit-exact CPU RNS-CKKS twin
             of the GPU product (parity of ciphertexts)
  _ref/      the reference itself, compiled from /root/reference by ref.mk
"""
