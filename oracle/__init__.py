"""CPU oracle for the FCM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import anything from this package. The product path
(paper_2404_19331_b200/) never imports it and shares no code with it; both sides
only share the seeded input generators in synth/.

Modules
  numerics  rounding to the storage formats (RNE) and the int8 fixed-point requantiser
  conv      DW, PW, DWPW = PW(DW(X)), PWDW = DW(PW(X)) exactly as PAPER.md defines them
            ("one filter applied to a single channel" / "1x1 filters span over all
            channels"; P:94 each conv is followed by normalisation + activation; P:111 the
            intermediate is held in the feature-map dtype; P:144 int8 results are packed
            (i.e. requantised to int8) before being written to ANY buffer)
  counting  FusePlanner's memory-access models, Eq. 1-4 verbatim, exact
            tile-enumeration counters, the fuse decision

Precision: floating point in float64, integer work in exact int64 / Python ints.
Parity status of every function is listed in DESIGN.md ("Oracle pins").
"""
