"""RelServe scheduling hot path, B200-native."""
