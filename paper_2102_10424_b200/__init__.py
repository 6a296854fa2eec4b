"""B200-native GIST hot path (arXiv 2102.10424): C-ABI library libgist.so + ctypes binding."""
from .gist import Gist, GistError, lib  # noqa: F401
