"""ctypes declarations of the task / reward entry points (filled in as they land)."""


def declare(lib):
    return lib
