"""B200-native time-stepping hot path for the ensemble MHD scheme of arXiv 2108.05110."""
