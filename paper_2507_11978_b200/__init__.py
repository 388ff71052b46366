"""B200-native backend for the NineToothed kernel set (arXiv 2507.11978)."""
