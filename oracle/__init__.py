"""ORACLE / TEST INFRASTRUCTURE — never imported by the product package.

`oracle.rank1_oracle` is our CPU restatement of the reference hot path
(numpy + the plain-C core in rank1_oracle.c); `oracle.ref` binds the compiled,
unmodified reference (oracle/_ref/librank1_ref.so) through its C-ABI shim.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use them.
"""
