"""B200-native shape-coefficient path (placeholder; filled in below)."""
