"""simjoin-b200: B200-native cosine-threshold tensor join (hot path of
arXiv 2312.01476's context-enhanced join), drop-in for the reference
``simjoin`` package's join/embedding API."""

__version__ = "0.1.0"
