"""B200-native single-pulse search hot path (Heimdall++ / pulsegrid drop-in)."""
