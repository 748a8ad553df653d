"""TEST INFRASTRUCTURE ONLY: the CPU oracle (see oracle/splat_oracle.hpp)."""
