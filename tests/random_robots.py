"""Random serial-chain URDFs for parity tests: interleaved fixed joints, random
origins (xyz + rpy), random unit axes, revolute / continuous / prismatic joints
and an optional mimic joint -- the shapes `compile_chain` must fold correctly."""

import numpy as np


def random_chain_urdf(seed: int, n_act: int = 7, fixed_every: int = 2, prismatic: bool = True,
                      mimic: bool = True) -> str:
    rng = np.random.default_rng(seed)
    links = ["base"]
    joints = []
    act = 0
    idx = 0
    mimic_src = None
    while act < n_act:
        idx += 1
        parent, child = links[-1], f"l{idx}"
        links.append(child)
        xyz = rng.uniform(-0.15, 0.15, 3) + np.array([0.0, 0.0, 0.12])
        rpy = rng.uniform(-np.pi, np.pi, 3)
        org = f'<origin xyz="{xyz[0]:.6f} {xyz[1]:.6f} {xyz[2]:.6f}" rpy="{rpy[0]:.6f} {rpy[1]:.6f} {rpy[2]:.6f}"/>'
        if fixed_every and idx % (fixed_every + 1) == 0:
            joints.append(f'<joint name="f{idx}" type="fixed"><parent link="{parent}"/><child link="{child}"/>{org}'
                          f'</joint>')
            continue
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        axis = f'<axis xyz="{ax[0]:.6f} {ax[1]:.6f} {ax[2]:.6f}"/>'
        kind = "revolute"
        if prismatic and act == 2:
            kind = "prismatic"
        elif act == 4:
            kind = "continuous"
        lim = {"revolute": '<limit lower="-2.6" upper="2.6" effort="1" velocity="2"/>',
               "prismatic": '<limit lower="-0.2" upper="0.3" effort="1" velocity="0.5"/>',
               "continuous": '<limit effort="1" velocity="3"/>'}[kind]
        joints.append(f'<joint name="j{act}" type="{kind}"><parent link="{parent}"/><child link="{child}"/>{org}'
                      f'{axis}{lim}</joint>')
        if act == 1:
            mimic_src = f"j{act}"
        act += 1
        if mimic and act == 3 and mimic_src:
            idx += 1
            parent, child = links[-1], f"m{idx}"
            links.append(child)
            ax2 = rng.normal(size=3)
            ax2 /= np.linalg.norm(ax2)
            joints.append(f'<joint name="mim{idx}" type="revolute"><parent link="{parent}"/><child link="{child}"/>'
                          f'<origin xyz="0.05 0.02 0.1" rpy="0.3 -0.2 0.5"/>'
                          f'<axis xyz="{ax2[0]:.6f} {ax2[1]:.6f} {ax2[2]:.6f}"/>'
                          f'<limit lower="-2" upper="2" effort="1" velocity="1"/>'
                          f'<mimic joint="{mimic_src}" multiplier="-0.7" offset="0.25"/></joint>')
    idx += 1
    links.append("tool")
    joints.append(f'<joint name="tool_fixed" type="fixed"><parent link="{links[-2]}"/><child link="tool"/>'
                  f'<origin xyz="0.02 -0.03 0.11" rpy="0.1 0.2 -0.3"/></joint>')
    body = "".join(f'<link name="{l}"/>' for l in links) + "".join(joints)
    return f'<robot name="rand{seed}">{body}</robot>'
