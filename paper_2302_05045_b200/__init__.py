"""SAMO per-step parameter-state path, B200-native (sm_100a)."""
