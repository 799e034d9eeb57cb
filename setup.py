"""Build hook: compile liblq.so for sm_100a (nvcc) before the package is
copied, so an install carries the library.  Plain `python -m
paper_2404_08867_b200._build` does the same for an in-tree checkout."""

import importlib.util
import os

from setuptools import setup
from setuptools.command.build_py import build_py

HERE = os.path.dirname(os.path.abspath(__file__))


class BuildWithLibrary(build_py):
    def run(self):
        spec = importlib.util.spec_from_file_location(
            "lq_build", os.path.join(HERE, "paper_2404_08867_b200", "_build.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.build_native(verbose=True)
        super().run()


setup(cmdclass={"build_py": BuildWithLibrary})
