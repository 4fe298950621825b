"""TEST INFRASTRUCTURE: CPU oracle of the reference Louver path (see louver_oracle.h)."""
