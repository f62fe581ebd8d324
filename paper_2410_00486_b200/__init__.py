"""B200-native CaRtGS mapping hot path (placeholder, filled below)."""
