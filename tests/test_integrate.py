"""The reference-side binding: install/uninstall patch exactly the call sites."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources only exist in the build container")
def test_install_points_every_reference_call_site_at_the_gpu_path():
    sys.path.insert(0, REF)
    try:
        import pipesched
        from pipesched import cache, heuristics, listsched
        from paper_2510_05186_b200 import integrate
        cpu = listsched.run_order
        integrate.install(pipesched)
        try:
            for mod in (listsched, heuristics, cache, pipesched):
                assert mod.run_order is not cpu
                assert "GPU" in mod.run_order.__doc__
        finally:
            integrate.uninstall(pipesched)
        for mod in (listsched, heuristics, cache, pipesched):
            assert mod.run_order is cpu
    finally:
        sys.path.remove(REF)
