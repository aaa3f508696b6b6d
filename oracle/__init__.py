"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the update phase.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import anything under oracle/.  It is the checker,
never the product: the product path (paper_2410_21316_b200) never imports it.

Pinning: tests/test_oracle_pin.py checks every function here against golden
fixtures produced by running the reference package itself
(tests/golden/make_goldens.py imports /root/reference/pkg/src/optistate).
"""
