"""B200-native IMEX-DG hot path."""
