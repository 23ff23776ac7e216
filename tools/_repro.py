import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"]); sys.path.insert(0, os.path.join(os.environ["GRAFT_REPO_ROOT"], "tests"))
import pytest
sys.exit(pytest.main(["-x", "-q", "--tb=short", "-p", "no:cacheprovider", "-s",
                      "tests/test_full_configs.py::test_c4_heat_steps_bitwise_vs_oracle",
                      "tests/test_api_edges.py"]))
