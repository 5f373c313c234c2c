# TEST INFRASTRUCTURE ONLY -- the reference's own unit tests as checkers of
# the B200 C++ API.  Compiles proj/tests/test_{iq_transform,lls,hybrid_nn,
# fused,eval,channel_sim}.cpp UNMODIFIED, read where they lie under
# /root/reference (nothing is copied into the repo), against the reference's
# headers, the doctest subset and Eigen subset in paper_2206_05998_b200/host,
# and libnoma_host.so (the product: every compute call goes to the GPU).
# Outputs go to oracle/_ref/reftests/ only: git-ignored, but shipped to the
# GPU box with the repo snapshot, where tests/test_gpu_reference_suite.py
# runs them.  Without /root/reference this does nothing.
REF ?= /root/reference/proj
HERE := $(abspath .)
PKG := $(abspath ../paper_2206_05998_b200)
HOST := $(PKG)/host
OUT := $(HERE)/_ref/reftests
TESTS := iq_transform lls hybrid_nn fused eval channel_sim
CXX ?= g++
# the reference build's flags (CMakeLists.txt:27): -O3, no FMA contraction
CXXFLAGS = -O3 -std=c++20 -ffp-contract=off -w -I$(HOST)/doctest -I$(HOST)/eigen -I$(REF)/include -I$(REF)/tests

ifneq ($(wildcard $(REF)/tests/test_lls.cpp),)
all: $(TESTS:%=$(OUT)/test_%)
else
all:
	@echo "reftests: $(REF) absent, nothing to build"
endif

$(OUT)/test_%: $(REF)/tests/test_%.cpp $(PKG)/libnoma_host.so $(HOST)/doctest/doctest.h $(wildcard $(HOST)/eigen/Eigen/*)
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(PKG) -lnoma_host -lnoma_b200 -Wl,-rpath,'$$ORIGIN/../../../paper_2206_05998_b200'

clean:
	rm -rf $(OUT)

.PHONY: all clean
