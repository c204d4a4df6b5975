"""CPU oracle for the hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import anything under oracle/.  It shares no
code with the CUDA path (paper_2405_14642_b200/) and never imports it.
"""
