"""B200-native (sm_100a) structure-preserving Bethe-Salpeter eigensolver."""
__version__ = "0.1.0"
