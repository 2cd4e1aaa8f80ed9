"""Independent exactness checkers (fp64, plain Python) that pin the oracle.

They implement the closed forms / textbook definitions the method reduces to in special
cases (SURVEY.md §8(c) "Pins"): brute-force alignment enumeration, the CTC forward
algorithm (Graves et al. 2006, PAPER.md ref [4]), greedy CTC decoding, the standard ARPA
backoff recursion and an Aho-Corasick booster. None of them imports the oracle or the
CUDA product.
"""
