# TEST INFRASTRUCTURE ONLY — builds the reference implementation itself into
# oracle/_ref/ (git-ignored; travels to the GPU box with the snapshot):
#   libhodlrgp_ref.so  the reference's hot-path sources, compiled UNMODIFIED from
#                      /root/reference/proj/src against the Eigen-API shim
#                      (oracle/eigen_shim), plus the or_* C ABI (ref_capi.cpp)
#                      that pyoracle binds — the parity oracle / CPU baseline;
#   ref_unit_tests     the reference's own doctest suites (proj/tests/test_*.cpp,
#                      unmodified) over the same objects, with the doctest shim.
# Nothing is copied out of /root/reference; sources are read where they lie.
# Usage: make -f ref.mk   (a no-op when /root/reference is absent)
REF ?= /root/reference/proj
CXX := /usr/bin/g++
OUT := _ref
# Same flags as the restated oracle (no FMA contraction, like the reference's
# default x86-64 build; -fvisibility=hidden keeps the C++ symbols private so
# this library and liboracle.so can be loaded side by side).
CXXFLAGS := -O3 -march=x86-64-v3 -ffp-contract=off -fopenmp -fPIC -std=c++20 -fvisibility=hidden \
            -Ieigen_shim -I$(REF)/include -I.
LIBSRC := cluster_tree hodlr_matrix sketch factorization product_rep mle
MODSRC := nonstationary1d simulate
TESTS := cluster_tree hodlr_matrix sketch factorization product_rep mle main
LIBOBJ := $(LIBSRC:%=$(OUT)/obj/src_%.o) $(OUT)/obj/shim.o $(OUT)/obj/dense.o
MODOBJ := $(MODSRC:%=$(OUT)/obj/model_%.o)
TESTOBJ := $(TESTS:%=$(OUT)/obj/test_%.o)
SHIM_HDR := eigen_shim/Eigen/Dense

ifeq ($(wildcard $(REF)/src/sketch.cpp),)
all:
	@echo "ref.mk: $(REF) not present; using the prebuilt oracle/_ref (if any)"
else
all: $(OUT)/libhodlrgp_ref.so $(OUT)/ref_unit_tests
endif

$(OUT)/obj/src_%.o: $(REF)/src/%.cpp $(SHIM_HDR)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@
$(OUT)/obj/model_%.o: $(REF)/src/models/%.cpp $(SHIM_HDR)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@
$(OUT)/obj/test_%.o: $(REF)/tests/test_%.cpp $(SHIM_HDR) doctest_shim/doctest.h
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -Idoctest_shim -c $< -o $@
$(OUT)/obj/shim.o: eigen_shim/shim.cpp $(SHIM_HDR) oracle.hpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@
$(OUT)/obj/dense.o: dense.cpp oracle.hpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@
$(OUT)/obj/ref_capi.o: ref_capi.cpp matern1d.hpp $(SHIM_HDR)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libhodlrgp_ref.so: $(LIBOBJ) $(OUT)/obj/ref_capi.o
	$(CXX) -shared -fopenmp -o $@ $^ -ldl
$(OUT)/ref_unit_tests: $(TESTOBJ) $(LIBOBJ) $(MODOBJ)
	$(CXX) -fopenmp -o $@ $^ -ldl

clean:
	rm -rf $(OUT)
.PHONY: all clean
