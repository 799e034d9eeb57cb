"""latquad.cli -> paper_2404_08867_b200.cli."""
from paper_2404_08867_b200.cli import *  # noqa: F401,F403
from paper_2404_08867_b200.cli import cli_main, main  # noqa: F401

if __name__ == "__main__":
    raise SystemExit(main())
