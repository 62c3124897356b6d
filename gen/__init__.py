from .gen import Generator, PRESETS  # noqa: F401
