"""pytest plugin (``-p ref_seam_plugin``) for running the REFERENCE's own test
files with its solver seam bound to the B200 library -- TEST INFRASTRUCTURE.
The reference package must be importable (baseline/_ref on PYTHONPATH)."""


def pytest_configure(config):
    import fftcond

    import ref_seam

    ref_seam.install(fftcond)
    config.addinivalue_line("markers", "b200_seam: reference tests through the B200 seam")
