"""latquad.corpus -> paper_2404_08867_b200.corpus."""
from paper_2404_08867_b200.corpus import *  # noqa: F401,F403
from paper_2404_08867_b200.corpus import CorpusEntry, all_ids, corpus_expr, entries, get, reference_value  # noqa: F401
