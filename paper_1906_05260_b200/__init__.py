"""B200-native VIPER rod-solver substep (arXiv 1906.05260) behind the reference's C++ core API."""
