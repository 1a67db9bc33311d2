"""CPU oracle for the Chimera scheduling-tick hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's `cpu_baseline` /
`--impl reference` legs may import this package, and only as the checker or
as the timed CPU reference arm. The product path (paper_2603_22206_b200) never
imports it and has no CPU fallback.

Contents
  hetsched_port.py  pure-Python restatement of the reference path
                    (hetsched.balancer/monitor/predictor/engine), same
                    algorithm and same cost structure (dict re-sum per
                    decision, lazy-deletion heap), each function citing the
                    reference file:line it follows.
  trace_ref.py      numpy restatement of TraceRecord.remaining_tokens and
                    first/next_stage_request on dense trace columns.
  encoder_ref.py    torch fp32 restatement of the router encoder (the
                    reference has no neural router: router.py only pins the
                    contract -- one score per pool model in [0,1]).

Parity pinning: hetsched_port is checked against golden vectors produced by
running the unmodified reference (/root/reference/pkg/src/hetsched) in the
build container -- tests/golden/make_golden.py writes them, tests/test_oracle.py
checks them -- and, when /root/reference is present, against the reference
itself on randomized inputs (tests/test_oracle_vs_reference.py).
"""
