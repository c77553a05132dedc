"""BENCH/TEST INFRASTRUCTURE -- seeded synthetic inputs (not part of the
aligner product in paper_2303_01845_b200/).

  workloads  BASELINE configs 2, 3, 5 as lists of byte strings (numpy) and,
             much faster, as a packed arena + pair table (C, gen.c)
  corpus     the reference's synthetic FASTA corpora (configs 1 and 4)
"""
