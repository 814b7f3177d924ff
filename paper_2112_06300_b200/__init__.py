"""B200-native conservative CCD (arXiv 2112.06300) — see DESIGN.md."""
