"""TEST INFRASTRUCTURE ONLY — CPU checkers for the B200 assembly path.

``oracle.port``  ctypes binding of our plain-C restatement (oracle/tg_oracle.c)
``oracle.ref``   ctypes binding of the unmodified reference library compiled
                 from /root/reference (oracle/_ref/libtgref.so, via ref_shim.cpp)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never on the product path.
"""
