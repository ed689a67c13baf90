"""CPU ORACLE for the EP-HDC client-side inference hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import or execute anything in this package.  The product
path (paper_2511_00737_b200) never imports it; the two share no code.  The only
common module is ephdc_inputs (seeded raw inputs, no method arithmetic).

What it computes, from PAPER.md (citations are "P:<line>"):
  * random-projection HDC encoding and quantisation;
  * single-pass training = bundling of encoded samples;
  * BFV with SIMD batching: slot encode = inverse negacyclic
    NTT mod t, symmetric encryption of the k-interleaved class HVs as D
    ciphertexts;
  * the client evaluation sum_d CT_d * PT_d: D MulCP, D-1 AddCC, 0 rotations
    (P:606-607);
  * decryption / decoding and argmax.

Everything here is plain: textbook loops, __int128 "(a*b) % q" products,
Python big integers for the CRT.  Every function is pinned in tests/ against
closed forms, brute force or the paper.
"""
