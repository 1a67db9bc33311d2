"""Synthetic workloads for the benchmark and the parity tests -- NOT part of the
product package (paper_2603_22206_b200).

  tracegen.py  draw-for-draw restatement of hetsched's synthetic trace
               generator and request types (workload.py:87-495), so the
               synthetic ticks match what the reference would generate
  synth.py     BASELINE.json's five configurations as seeded workloads
               (pool, router weights, predictor, batches, pre-tick state)
"""
