"""B200-native hybrid AB-/BA-GMRES projector path."""
