// Force-included (-include) when oracle/Makefile compiles the reference's UNMODIFIED acceptance suite
// (proj/tests/acceptance.cpp) for the B200 backend: its training calls resolve to the transport.backend = "b200"
// entry points of integration/b200_backend.cpp. The macros also rename the two declarations in
// lsgd/executors.hpp, which therefore declare exactly the functions b200_backend.cpp defines.
#pragma once
#define run_train run_train_b200
#define verify_equivalence verify_equivalence_b200
