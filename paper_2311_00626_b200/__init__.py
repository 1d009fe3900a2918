"""B200-native per-frame map update (nvblox / voxmap hot path)."""
