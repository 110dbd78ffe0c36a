"""B200-native RAC-MBADMM sweep (arXiv 1907.01995) behind the racml entry points."""
