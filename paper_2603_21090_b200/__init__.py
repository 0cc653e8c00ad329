"""B200-native StreamTGN incremental inference path."""
