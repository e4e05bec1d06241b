"""B200-native GLMB step core (arXiv 2512.06230): predict, birth, compat, reweight."""
